"""The reference's own hot-path test sources (proj/tests/test_*.cpp), compiled
unmodified against our drop-in headers include/pulse/*.hpp + libpulse_cuda.so
(tests/cpp/Makefile; built by __graft_entry__.build() where /root/reference is
mounted, shipped prebuilt to the GPU box).  Suites that only touch host code
run on CPU; the rest drive the CUDA kernels and are GPU tests."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_bin")

HOST_SUITES = ["test_bf16", "test_compression", "test_hashing", "test_synthetic", "test_container"]
GPU_SUITES = ["test_patch", "test_index_coding", "test_patch_file", "test_metrics", "test_absorption"]


def _run(suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "All tests passed" in r.stdout


@pytest.mark.parametrize("suite", HOST_SUITES)
def test_reference_suite_host(suite):
    _run(suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_suite_gpu(suite):
    _run(suite)
