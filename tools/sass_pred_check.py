"""Scan the SASS of a built library for one ptxas 12.9 miscompile pattern found in f_pass:

    @P0 IADD3 R0, P0, PT, R6, R12, RZ    <- guarded by P0, writes the carry into P0
        ...
    @P0 STL [R1], R0                      <- still meant as the old guard, now reads the carry

i.e. an instruction guarded by Pk that also writes Pk, followed (before any other write of Pk)
by an instruction GUARDED by Pk.  Using Pk as a carry input (IMAD.X ..., Pk) is legitimate.
    python tools/sass_pred_check.py paper_2602_03839_b200/libpulse_cuda.so
Exit status 1 if any function matches."""
import re
import subprocess
import sys

so = sys.argv[1]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
ins_re = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?P([0-6])\s+)?([A-Z0-9_.]+)\s*([^;]*);")
bad = []
fn = None
pending = {}  # predicate -> (addr, text) of a guarded self-write still live
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn, pending = m.group(1), {}
        continue
    m = ins_re.search(line)
    if not m:
        continue
    addr, guard, gp, op, args = m.group(1), m.group(2), m.group(3), m.group(4), m.group(5)
    if op.startswith("BRA") or op in ("EXIT", "RET", "CALL", "BSYNC", "BSSY", "WARPSYNC"):
        pending = {}  # control flow: stop tracking (conservative)
        continue
    if gp is not None and gp in pending:
        bad.append((fn, pending[gp], f"{addr}: {line.strip()[:90]}"))
        del pending[gp]
    # predicate destinations: tokens P0..P6 among the leading outputs (before the first source)
    outs = [t.strip() for t in args.split(",")]
    written = set()
    for t in outs[:3]:
        if re.fullmatch(r"P[0-6]", t):
            written.add(t[1])
    uses_as_input = set(re.findall(r"\bP([0-6])\b", ",".join(outs[2:])))
    for p in written:
        pending.pop(p, None)
    if gp is not None and gp in written and op.startswith(("IADD3", "IMAD", "ISETP", "LOP3", "IADD")):
        pending[gp] = f"{addr}: {line.strip()[:90]}"
for fn_, a, b in bad:
    print(f"{fn_}\n  {a}\n  {b}")
print(f"{len(bad)} suspicious guarded predicate reuse(s) in {so}")
sys.exit(1 if bad else 0)
