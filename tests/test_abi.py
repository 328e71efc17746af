"""CPU checks of the C-ABI boundary: the library loads (no GPU needed) and
exports every function include/pulse_cuda.h declares."""
import os
import re
import subprocess

import pytest

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


def test_plain_c_consumer_compiles(tmp_path):
    """include/pulse_cuda.h is a C header: a C11 program using it builds warning-free."""
    import subprocess
    src = os.path.join(ROOT, "examples", "c_abi_roundtrip.c")
    out = tmp_path / "c_abi_roundtrip.o"
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-c", "-I", os.path.join(ROOT, "include"),
                        src, "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_plain_c_consumer_round_trip():
    import subprocess
    exe = os.path.join(ROOT, "tests", "_bin", "c_abi_roundtrip")
    if not os.path.exists(exe):
        pytest.skip("examples/c_abi_roundtrip not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "C ABI round trip OK" in r.stdout


@pytest.mark.skipif(not os.path.exists("/usr/local/cuda/bin/cuobjdump"), reason="needs cuobjdump")
def test_sass_has_no_guarded_predicate_clobber():
    """The shipped SASS is free of the ptxas 12.9 pattern that once left F3's range end stale
    (an add guarded by Pk that writes its carry into Pk, then a store still guarded by Pk)."""
    r = subprocess.run(["python", os.path.join(ROOT, "tools", "sass_pred_check.py"), LIB], capture_output=True,
                       text=True, env={**os.environ, "PATH": os.environ.get("PATH", "") + ":/usr/local/cuda/bin"})
    assert r.returncode == 0, r.stdout[-2000:]
