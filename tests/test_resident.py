"""Resident checkpoints: the sync path on the device (sync.hpp apply_delta /
walk_deltas / publish_checkpoint's patch) against the reference's own PULP
bytes (golden fixtures) and the reference itself (oracle/_ref) for chains."""
import numpy as np
import pytest

from oracle.oracle import IDENTITY, ZSTD1, have_reference, reference
from paper_2602_03839_b200 import host as H
from paper_2602_03839_b200._native import PulseError

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = ["roundtrip_s0", "patchfile_s1", "accept_b", "handcrafted", "esc_cols"]


def mirror(ck, step=None):
    return H.Checkpoint(ck.step if step is None else step, [H.Tensor(t.name, tuple(t.shape), t.data) for t in ck.tensors])


def same(a, b):
    return [(t.name, tuple(t.shape)) for t in a.tensors] == [(t.name, tuple(t.shape)) for t in b.tensors] and all(
        np.array_equal(x.data, y.data) for x, y in zip(a.tensors, b.tensors))


@pytest.mark.parametrize("repr_", [0, 1, 2])
@pytest.mark.parametrize("codec", [IDENTITY, ZSTD1])
def test_apply_reference_pulp(golden, repr_, codec):
    for name in CASES:
        prev, curr, m = golden.case(name)
        wire = golden.pulp(name, repr_, codec)
        if wire is None:
            continue
        r = H.Resident(mirror(prev), max_changes=1024)
        assert r.step == 0 and r.weights_hash == H.hash_weights(mirror(prev))
        r.apply(wire, 1, expected_hash=bytes.fromhex(m["target_hash"]), verify=True)
        assert r.step == 1 and r.weights_hash.hex() == m["target_hash"]
        assert same(r.download(), mirror(curr))


def test_protocol_and_model_errors(golden):
    prev, curr, m = golden.case("roundtrip_s1")
    wire = golden.pulp("roundtrip_s1", 0, IDENTITY)
    r = H.Resident(mirror(prev))
    for step, exp, kind in [(2, None, "ProtocolViolationError"),
                            (1, b"\1" * 32, "ProtocolViolationError")]:
        with pytest.raises(PulseError) as ei:
            r.apply(wire, step, expected_hash=exp)
        assert ei.value.kind == kind
    held = H.Resident(mirror(prev, step=5))       # base step 0 != held 5
    with pytest.raises(PulseError) as ei:
        held.apply(wire, 6)
    assert ei.value.kind == "ProtocolViolationError"
    other = H.Checkpoint(0, [H.Tensor("zzz", (3,), np.zeros(3, np.uint16))])
    with pytest.raises(PulseError) as ei:
        H.Resident(other).apply(wire, 1)
    assert ei.value.kind == "TensorSetError"
    reshaped = mirror(prev)
    t0 = reshaped.tensors[0]
    reshaped.tensors[0] = H.Tensor(t0.name, (t0.data.size,), t0.data)
    with pytest.raises(PulseError) as ei:
        H.Resident(reshaped).apply(wire, 1)
    assert ei.value.kind == "ShapeMismatchError"
    assert r.step == 0 and same(r.download(), mirror(prev))


def test_tampered_value_fails_hash_and_leaves_state(golden):
    """A value flipped inside the PULP (identity codec): the verified apply fails
    with HashMismatchError and the held weights, step and hash are unchanged."""
    prev, curr, m = golden.case("accept_b")
    wire = bytearray(golden.pulp("accept_b", 0, IDENTITY))
    wire[-1] ^= 0x40                                  # last value byte of the last tensor
    r = H.Resident(mirror(prev))
    h0 = r.weights_hash
    with pytest.raises(PulseError) as ei:
        r.apply(bytes(wire), 1, verify=True)
    assert ei.value.kind == "HashMismatchError"
    assert r.step == 0 and r.weights_hash == h0 and same(r.download(), mirror(prev))
    # corrupt index payload: the reference's exception, nothing written
    bad = bytearray(golden.pulp("accept_b", 1, IDENTITY))
    hl = int.from_bytes(bad[8:16], "little")
    bad[16 + hl:16 + hl + 4] = b"\xff\xff\xff\x7f"    # first u32: index far past the tensor
    with pytest.raises(PulseError) as ei:
        r.apply(bytes(bad), 1)
    assert ei.value.kind == "CorruptStreamError"
    assert r.step == 0 and same(r.download(), mirror(prev))


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
@pytest.mark.parametrize("repr_", [0, 2])
def test_walk_reference_chain(repr_):
    """walk_deltas over a chain the reference encoded (k = 5 steps)."""
    R = reference()
    base, _ = R.generate_synthetic([(64, 96), (1000,), (7, 11, 13)], 0.97, 16, 3)
    chain = [base]
    for k in range(5):
        chain.append(R.mutate(chain[-1], 0.98, 8, 100 + k, k + 1))
    wires = [R.write_patch_bytes(R.encode(chain[k + 1], chain[k], repr_, ZSTD1)) for k in range(5)]
    r = H.Resident(mirror(chain[0]))
    assert r.walk(wires, verify=True) == 5
    assert r.step == 5 and r.weights_hash == R.hash_weights(chain[5])
    assert same(r.download(), mirror(chain[5]))
    # a walk stops at the first failure and keeps what it applied
    r2 = H.Resident(mirror(chain[0]))
    bad = bytearray(wires[2])
    bad[0] = ord("X")
    with pytest.raises(PulseError):
        r2.walk([wires[0], wires[1], bytes(bad), wires[3]])
    assert r2.last_walk_applied == 2 and r2.step == 2 and same(r2.download(), mirror(chain[2]))


@pytest.mark.parametrize("repr_", [0, 1, 2])
@pytest.mark.parametrize("codec", [IDENTITY, ZSTD1])
def test_publish_matches_reference_pulp(golden, repr_, codec):
    """publish from device-resident weights: the PULP bytes equal the reference's
    write_patch_bytes(encode(curr, prev)) and the hash its hash_weights(curr);
    with advance the resident becomes the published snapshot, and a consumer
    resident applying those bytes lands on the same weights."""
    for name in CASES:
        prev, curr, m = golden.case(name)
        want = golden.pulp(name, repr_, codec)
        if want is None:
            continue
        pub = H.Resident(mirror(prev), max_changes=1024)
        cur_d = [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in curr.tensors]
        wire, h = pub.publish(cur_d, 1, repr_, codec, anchor_step=0, advance=True)
        assert wire == want, (name, repr_, codec)
        assert h.hex() == m["target_hash"]
        assert pub.step == 1 and pub.weights_hash == h and same(pub.download(), mirror(curr, 1))
        sub = H.Resident(mirror(prev))
        sub.apply(wire, 1, expected_hash=h)
        assert same(sub.download(), mirror(curr, 1))


def test_publish_requires_consecutive_steps(golden):
    prev, curr, _ = golden.case("roundtrip_s0")
    pub = H.Resident(mirror(prev))
    cur_d = [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in curr.tensors]
    with pytest.raises(PulseError) as ei:
        pub.publish(cur_d, 3)
    assert ei.value.kind == "ArgumentError"
    assert pub.step == 0 and same(pub.download(), mirror(prev))


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
def test_walk_stops_on_hash_mismatch_and_keeps_the_last_good_step():
    """A walk with verification over a chain whose third delta carries a tampered
    value (identity codec): steps 1-2 apply, step 3 fails with HashMismatchError,
    and the held weights, step and hash are exactly those of step 2."""
    R = reference()
    base, _ = R.generate_synthetic([(48, 32), (700,)], 0.96, 8, 5)
    chain = [base]
    for k in range(4):
        chain.append(R.mutate(chain[-1], 0.97, 8, 300 + k, k + 1))
    wires = [bytearray(R.write_patch_bytes(R.encode(chain[k + 1], chain[k], 0, IDENTITY))) for k in range(4)]
    wires[2][-1] ^= 0x01  # last value byte of the third delta
    r = H.Resident(mirror(chain[0]))
    with pytest.raises(PulseError) as ei:
        r.walk([bytes(w) for w in wires], verify=True)
    assert ei.value.kind == "HashMismatchError"
    assert r.last_walk_applied == 2 and r.step == 2
    assert r.weights_hash == R.hash_weights(chain[2]) and same(r.download(), mirror(chain[2]))
