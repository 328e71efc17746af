"""PULC checkpoint container (reference container.hpp) through the C ABI:
the writer's bytes against the reference's (SHA-256 pins in
tests/golden/containers.json, made by make_golden_pulc.py from the reference
itself), the reader's acceptance / exception class / message on damaged
containers, and the device-direct load and store paths (GPU)."""
import hashlib
import importlib.util
import json
import os

import numpy as np
import pytest

from oracle.oracle import Checkpoint as OCheckpoint, Tensor as OTensor
from paper_2602_03839_b200 import host as H
from paper_2602_03839_b200._native import PulseError

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "containers.json")) as _f:
    PULC = json.load(_f)
_spec = importlib.util.spec_from_file_location("make_golden_pulc", os.path.join(HERE, "golden", "make_golden_pulc.py"))
G = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(G)  # the shared case builders (never runs the reference)


def mirror(ck):
    return H.Checkpoint(ck.step, [H.Tensor(t.name, tuple(t.shape), t.data) for t in ck.tensors])


def snapshot(golden, name, side):
    prev, curr, _ = golden.case(name)
    return mirror(prev if side == "prev" else curr)


def test_writer_matches_reference_bytes(golden):
    for key, want in PULC["snapshots"].items():
        name, side = key.split("/")
        b = H.write_checkpoint_bytes(snapshot(golden, name, side))
        assert len(b) == want["nbytes"], key
        assert hashlib.sha256(b).hexdigest() == want["sha256"], key


def test_writer_handbuilt_edge_cases():
    for name, ck in G.handbuilt(OCheckpoint, OTensor).items():
        b = H.write_checkpoint_bytes(mirror(ck))
        want = PULC["handbuilt"][name]
        assert (len(b), hashlib.sha256(b).hexdigest()) == (want["nbytes"], want["sha256"]), name
        back = H.read_checkpoint_bytes(b)
        assert back.step == ck.step
        assert [(t.name, tuple(t.shape)) for t in back.tensors] == [(t.name, tuple(t.shape)) for t in ck.tensors]
        for a, t in zip(back.tensors, ck.tensors):
            assert np.array_equal(a.data, t.data)


def test_round_trip_and_alignment(golden):
    ck = snapshot(golden, "roundtrip_s0", "curr")
    b = H.write_checkpoint_bytes(ck)
    back = H.read_checkpoint_bytes(np.frombuffer(b, np.uint8))
    assert H.write_checkpoint_bytes(back) == b  # canonical
    c = H.Container(b)
    for _, _, _, off in c.tensors:
        assert off % 64 == 0
    assert H.hash_weights(back) == H.hash_weights(ck)


def test_reader_errors_match_reference():
    for label, data in G.corruptions():
        want = PULC["corruptions"][label]
        if want["status"] == 0:
            back = H.read_checkpoint_bytes(data)
            assert back.step == want["step"], label
            assert [[t.name, list(t.shape), t.data.tolist()] for t in back.tensors] == want["tensors"], label
            continue
        with pytest.raises(PulseError) as ei:
            H.read_checkpoint_bytes(data)
        assert ei.value.status == want["status"], (label, str(ei.value))
        assert str(ei.value) == want["message"], label


def test_writer_validates_like_reference():
    bad = H.Checkpoint(0, [H.Tensor("a", (2,), np.zeros(2, np.uint16)), H.Tensor("a", (1,), np.zeros(1, np.uint16))])
    with pytest.raises(PulseError) as ei:
        H.write_checkpoint_bytes(bad)
    assert ei.value.kind == "ArgumentError"


@pytest.mark.gpu
def test_device_load_and_store(golden):
    import torch

    for name in ("roundtrip_s1", "handcrafted", "accept_b"):
        ck = snapshot(golden, name, "curr")
        b = H.write_checkpoint_bytes(ck)
        dev = [torch.empty(t.data.size, dtype=torch.int16, device="cuda") for t in ck.tensors]
        c = H.read_checkpoint_to_device(b, dev)
        assert c.step == ck.step
        for d, t in zip(dev, ck.tensors):
            assert np.array_equal(d.cpu().numpy().view(np.uint16), t.data)
        back = H.write_checkpoint_bytes_from_device(ck.step, [t.name for t in ck.tensors],
                                                    [t.shape for t in ck.tensors], dev)
        assert back == b


@pytest.mark.gpu
def test_device_load_large_pinned_and_pageable():
    """A multi-chunk container (> the 64 MiB staging chunk) loaded from pageable
    bytes and from page-locked bytes lands bit-exact in HBM."""
    import torch

    rng = np.random.default_rng(3)
    shapes = [(4096, 5120), (3, 7), (11008, 4096)]
    ck = H.Checkpoint(9, [H.Tensor(f"t{i}", s, rng.integers(0, 65536, int(np.prod(s)), dtype=np.uint16))
                          for i, s in enumerate(shapes)])
    b = H.write_checkpoint_bytes(ck)
    pinned = torch.empty(len(b), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(b, np.uint8)
    for src in (b, pinned.numpy()):
        dev = [torch.empty(t.data.size, dtype=torch.int16, device="cuda") for t in ck.tensors]
        H.read_checkpoint_to_device(src, dev)
        for d, t in zip(dev, ck.tensors):
            assert torch.equal(d.cpu(), torch.from_numpy(t.data.view(np.int16)))
    out = H.write_checkpoint_bytes_from_device(ck.step, [t.name for t in ck.tensors], shapes, dev)
    assert out == b


@pytest.mark.gpu
def test_device_paths_reject_bad_pointers():
    import torch

    ck = H.Checkpoint(1, [H.Tensor("w", (4,), np.arange(4, dtype=np.uint16))])
    b = H.write_checkpoint_bytes(ck)
    with pytest.raises(PulseError):
        H.read_checkpoint_to_device(b, [torch.empty(3, dtype=torch.int16, device="cuda")])
    host_t = torch.zeros(4, dtype=torch.int16)
    with pytest.raises(PulseError) as ei:
        H.write_checkpoint_bytes_from_device(1, ["w"], [(4,)], [host_t])
    assert ei.value.kind == "ArgumentError"
