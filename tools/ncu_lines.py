"""Attribute an ncu SASS source export (ncu --page source --csv --print-source sass)
to CUDA source lines using `nvdisasm -g` of the same object: stall samples and
executed warp-instructions per file:line.
Usage: python tools/ncu_lines.py export.csv disasm.sass mangled_kernel_name [top]"""
import collections
import csv
import re
import sys


def main():
    path, sass, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(path)))
    h = rows[1]
    iA, iS, iX, iW = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                           "Warp Stall Sampling (All Samples)"))
    recs = [(int(r[iA], 16), r[iS].strip(), int(r[iX] or 0), int(r[iW] or 0))
            for r in rows[2:] if len(r) > iW and r[iA].startswith("0x")]
    base = recs[0][0]
    lines = open(sass).read().split("\n")
    start = [i for i, l in enumerate(lines) if l.startswith(".text." + kname + ":")][0]
    cur, off2line = None, {}
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(\S.*?);", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    agg, ex = collections.Counter(), collections.Counter()
    for a, s, x, w in recs:
        ln = off2line.get(a - base)
        agg[ln] += w
        ex[ln] += x
    tot, totx = sum(r[3] for r in recs), sum(r[2] for r in recs)
    print(f"samples {tot}  executed warp-instructions {totx}")
    for k, v in sorted(agg.items(), key=lambda t: -t[1])[:top]:
        print(f"{v:7d} {v / max(tot, 1):6.1%} {ex[k]:11d} {ex[k] / max(totx, 1):6.1%} {k}")


if __name__ == "__main__":
    main()
