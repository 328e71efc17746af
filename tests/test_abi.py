"""CPU checks of the C-ABI boundary: the library loads (no GPU needed) and
exports every function include/pulse_cuda.h declares."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pulse_cuda.h")
LIB = os.path.join(ROOT, "paper_2602_03839_b200", "libpulse_cuda.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pulse_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("pulse_encode_scan", "pulse_encode_emit", "pulse_apply", "pulse_plan_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (pulse_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_resolves():
    from paper_2602_03839_b200 import _native as N
    assert N.lib.pulse_version().startswith(b"pulse-b200")
    for name in declared():
        assert hasattr(N.lib, name)
