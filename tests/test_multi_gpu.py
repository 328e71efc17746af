"""Multi-GPU (N >= 2 devices on one box, NCCL): the sharded encode gathered to rank 0
over NCCL point-to-point (shard.gather) equals the single-GPU patch body and the
reference's (tools/check_shard.py under torchrun).  Skipped on a one-GPU box; the
one-GPU N-rank simulation in test_parity_configs.py covers the section logic there."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_sharded_gather_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29613", os.path.join(ROOT, "tools", "check_shard.py"),
           "qwen2.5-1.5b"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "CHECK_SHARD PASS" in r.stdout, r.stdout[-2000:]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_sharded_bench_step_two_ranks():
    """The device-side sharded step (K1 -> K2 -> size table over NVLink peer stores -> apply),
    captured as CUDA graphs: the weights land on the target and every rank's size row arrives."""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29614", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "qwen2.5-1.5b", "--steps", "4", "--warmup", "3", "--no-e2e",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["verified"] and line["config"]["launch"] == "cuda-graph replay", line


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_flat_summaries_over_nvlink_two_ranks():
    """FLAT_INT32 sharded step with the scan summaries all-gathered over NVLink inside the
    graph (pulse_peer_allgather, epoch-tagged slots): the FLAT carry it feeds must make every
    rank's apply land on the target."""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29615", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "qwen2.5-1.5b", "--repr", "2", "--steps", "4", "--warmup", "3",
           "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={k: v for k, v in os.environ.items() if k != "PULSE_PEER_SUMMARIES"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["verified"] and line["config"]["launch"] == "cuda-graph replay", line
    assert "NVLink summary table unavailable" not in r.stderr
