import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    """The reference-generated fixtures (tests/golden/make_golden.py)."""
    from oracle.oracle import Checkpoint, Tensor

    with open(os.path.join(GOLDEN, "golden.json")) as f:
        manifest = json.load(f)
    snaps = np.load(os.path.join(GOLDEN, "synth_cases.npz"))
    patches = np.load(os.path.join(GOLDEN, "patches.npz"))

    def case(name):
        m = manifest["cases"][name]
        shapes = [tuple(s) for s in m["shapes"]]
        prev = Checkpoint(0, [Tensor(n, s, snaps[f"{name}/prev/{i}"]) for i, (n, s) in enumerate(zip(m["names"], shapes))])
        curr = Checkpoint(1, [Tensor(n, s, snaps[f"{name}/curr/{i}"]) for i, (n, s) in enumerate(zip(m["names"], shapes))])
        return prev, curr, m

    def pulp(name, repr_, codec):
        key = f"{name}/{repr_}/{codec}"
        return patches[key].tobytes() if key in patches.files else None

    class G:
        pass

    g = G()
    g.manifest = manifest
    g.case = case
    g.pulp = pulp
    g.names = sorted(manifest["cases"])
    return g
