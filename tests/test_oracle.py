"""Pins the CPU oracle (oracle/pulse_oracle.c + oracle/oracle.py) before it is
trusted as the checker for the CUDA path.

* Known-answer vectors: the hand-computed bytes in the reference's own tests
  (proj/tests/test_index_coding.cpp, test_patch.cpp, test_hashing.cpp).
* Golden fixtures: outputs of the reference itself (tests/golden/, written by
  tests/golden/make_golden.py from oracle/_ref/libpulse_ref.so).
* Where the reference .so is present, randomized cross-checks against it.
"""
import numpy as np
import pytest

from oracle.oracle import (COO_DOWNSCALED, COO_INT32, FLAT_INT32, IDENTITY, Checkpoint, OracleError,
                           Patch, Tensor, TensorPatch, have_reference, reference, restatement)

S = restatement()
needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")


# ---- known-answer vectors from the reference's tests ---------------------------------------
def test_gap_encoding_kat():  # test_index_coding.cpp:32-41
    assert S.delta_encode([3, 5, 9, 100]).tolist() == [3, 2, 4, 91]
    assert S.delta_encode([0]).tolist() == [0]
    assert S.delta_encode([]).size == 0 and S.delta_decode([]).size == 0


def test_gap_encoding_rejects():  # test_index_coding.cpp:54-64
    for bad in ([3, 3], [5, 2], [-1, 2]):
        with pytest.raises(OracleError) as e:
            S.delta_encode(bad)
        assert e.value.kind == "ArgumentError"
    for bad in ([5, 0], [5, -2], [-3]):
        with pytest.raises(OracleError) as e:
            S.delta_decode(bad)
        assert e.value.kind == "FormatError"


def test_downscaled_kat():  # test_index_coding.cpp:66-79
    p = S.downscale_coo([0, 0, 2], [1, 3, 10])
    assert p == bytes([0x00, 0x00, 0x02, 0x01, 0x00, 0x02, 0x00, 0x0A, 0x00])
    r, c = S.upscale_coo(p, 3)
    assert r.tolist() == [0, 0, 2] and c.tolist() == [1, 3, 10]


def test_downscaled_escape_kat():  # test_index_coding.cpp:81-106
    assert S.downscale_coo([300], [70000]) == bytes([0xFF, 0x2C, 1, 0, 0, 0xFF, 0xFF, 0x70, 0x11, 1, 0])
    p = S.downscale_coo([0, 255], [65535, 7])
    assert len(p) == (1 + 5) + (6 + 2)
    r, c = S.upscale_coo(p, 2)
    assert r.tolist() == [0, 255] and c.tolist() == [65535, 7]


def test_downscaled_rejects():  # test_index_coding.cpp:168-197
    for rows, cols in (([0, 1], [0]), ([1, 0], [0, 0]), ([0, 0], [4, 4]), ([-1], [0])):
        with pytest.raises(OracleError) as e:
            S.downscale_coo(rows, cols)
        assert e.value.kind == "ArgumentError"
    p = S.downscale_coo([0, 0, 2], [1, 3, 10])
    with pytest.raises(OracleError) as e:
        S.upscale_coo(p[:-1], 3)
    assert e.value.kind == "TruncationError"
    with pytest.raises(OracleError) as e:
        S.upscale_coo(p + b"\0", 3)
    assert e.value.kind == "CorruptStreamError"
    with pytest.raises(OracleError) as e:
        S.upscale_coo(bytes([0, 0, 5, 0, 0, 0]), 2)
    assert e.value.kind == "CorruptStreamError"


def test_byte_accounting_random():  # test_index_coding.cpp:108-158
    rng = np.random.default_rng(0xC00C00)
    for _ in range(50):
        nr, nc, n = int(rng.integers(1, 2000)), int(rng.integers(1, 200000)), int(rng.integers(1, 400))
        flat = np.unique(rng.integers(0, nr * nc, n))
        rows, cols = flat // nc, flat % nc
        p = S.downscale_coo(rows, cols)
        r2, c2 = S.upscale_coo(p, rows.size)
        assert (r2 == rows).all() and (c2 == cols).all()
        rg = np.diff(rows, prepend=0)
        rg[0] = rows[0]
        new_row = np.ones(rows.size, bool)
        new_row[1:] = rows[1:] != rows[:-1]
        ce = np.where(new_row, cols, cols - np.concatenate([[0], cols[:-1]]))
        esc = int((rg >= 0xFF).sum() + (ce >= 0xFFFF).sum())
        assert len(p) == 3 * rows.size + 4 * esc


def test_int32_payload_kat():  # test_patch.cpp:200-214
    p = Patch(representation=COO_INT32, tensors=[TensorPatch("w", (128,), np.array([3, 5, 9, 100]), np.zeros(4, np.uint16))])
    assert S.encode_index_payloads(p) == [bytes([3, 0, 0, 0, 2, 0, 0, 0, 4, 0, 0, 0, 91, 0, 0, 0])]


def test_flat_gaps_cross_tensors_kat():  # test_patch.cpp:216-243
    p = Patch(representation=FLAT_INT32, tensors=[
        TensorPatch("a", (4,), np.array([1, 3]), np.zeros(2, np.uint16)),
        TensorPatch("b", (4,), np.array([0, 2]), np.zeros(2, np.uint16))])
    pl = S.encode_index_payloads(p)
    assert pl == [bytes([1, 0, 0, 0, 2, 0, 0, 0])] * 2
    back = S.decode_index_payloads(FLAT_INT32, [(4,), (4,)], [2, 2], pl)
    assert back[0].tolist() == [1, 3] and back[1].tolist() == [0, 2]


def test_downscaled_2d_view_kat():  # test_patch.cpp:245-264
    p = Patch(representation=COO_DOWNSCALED, tensors=[TensorPatch("w", (3, 4), np.array([1, 3, 10]), np.zeros(3, np.uint16))])
    pl = S.encode_index_payloads(p)
    assert pl == [S.downscale_coo([0, 0, 2], [1, 3, 2])]
    assert S.decode_index_payloads(COO_DOWNSCALED, [(3, 4)], [3], pl)[0].tolist() == [1, 3, 10]


@pytest.mark.parametrize("payload,kind", [
    (bytes([3, 0, 0, 0, 0, 0, 0, 0]), "CorruptStreamError"),   # zero gap
    (bytes([3, 0, 0, 0, 9, 0, 0, 0]), "CorruptStreamError"),   # out of range
    (bytes([3, 0, 0, 0, 1, 0, 0, 0, 7]), "CorruptStreamError"),  # trailing
    (bytes([3, 0, 0]), "TruncationError"),
])
def test_corrupt_int32_payloads(payload, kind):  # test_patch.cpp:266-294
    with pytest.raises(OracleError) as e:
        S.decode_index_payloads(COO_INT32, [(8,)], [2], [payload])
    assert e.value.kind == kind


def test_single_change_kat():  # test_patch.cpp:67-79  (3.5 in bf16 = 0x4060)
    prev = Checkpoint(0, [Tensor("w", (4,), np.array([0x3F80, 0x4000, 0x4040, 0x4080], np.uint16))])
    curr = Checkpoint(1, [Tensor("w", (4,), np.array([0x3F80, 0x4000, 0x4060, 0x4080], np.uint16))])
    p = S.encode(curr, prev)
    assert len(p.tensors) == 1 and p.tensors[0].indices.tolist() == [2] and p.tensors[0].values.tolist() == [0x4060]
    out = S.decode(prev, p)
    assert (out.tensors[0].data == curr.tensors[0].data).all()


def test_sha256_fips_vectors():  # test_hashing.cpp:44-54
    assert S.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert S.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert S.sha256(b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq").hex() == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"
    assert S.sha256(b"a" * 1000000).hex() == "cdc76e5c9914fb9281a1c7e284d73e67f1809a48a497200e046d39ccc7112cd0"


def test_hash_weights_name_order():  # test_hashing.cpp:27-40,73-94
    ck = Checkpoint(3, [Tensor("beta", (2, 2), np.array([0x3F80, 1, 0x8000, 0x7F7F], np.uint16)),
                        Tensor("alpha", (3,), np.array([0x4000, 0x4040, 0xC000], np.uint16))])
    canon = ck.tensors[1].data.tobytes() + ck.tensors[0].data.tobytes()
    assert S.hash_weights(ck) == S.sha256(canon)
    assert S.hash_weights(Checkpoint(0, [])).hex().startswith("e3b0c442")


# ---- golden fixtures produced by the reference ----------------------------------------------
def test_restatement_matches_golden_patches(golden):
    for name in golden.names:
        prev, curr, m = golden.case(name)
        assert S.hash_weights(curr).hex() == m["target_hash"]
        for r in (COO_DOWNSCALED, COO_INT32, FLAT_INT32):
            want = golden.pulp(name, r, IDENTITY)
            p = S.encode(curr, prev, r, IDENTITY)
            if want is None:
                continue
            assert S.write_patch_bytes_identity(p) == want, (name, r)
            # decode side: payloads parsed back to the same indices, apply rebuilds curr
            pl = S.encode_index_payloads(p)
            back = S.decode_index_payloads(r, [tp.shape for tp in p.tensors], [tp.indices.size for tp in p.tensors], pl)
            for b, tp in zip(back, p.tensors):
                assert (b == tp.indices).all()
            out = S.decode(prev, p)
            for a, b in zip(out.tensors, curr.tensors):
                assert (a.data == b.data).all()


def test_golden_config1_summary(golden):
    c1 = golden.manifest["config1"]
    assert c1["changes"] == 167772
    assert c1["target_hash"] == "903953d7d7a2fe189a4c074363a032ee4f9d713f4dc551f0de9a662bb3bf6325"
    assert c1["pulp_nbytes"]["0/0"] == 839187


def test_handcrafted_fixture_hits_escape_payload_markers(golden):
    prev, curr, _ = golden.case("handcrafted")
    p = S.encode(curr, prev, COO_DOWNSCALED, IDENTITY)
    pl = S.encode_index_payloads(p)
    assert bytes([0xFF, 0xFF, 0, 0, 0]) in pl[0]          # row gap 255 collides with the marker
    assert bytes([0xFF, 0xFF, 0xFF, 0xFF, 0, 0]) in pl[1]  # col entry 65535 -> FFFF + FFFF0000


# ---- randomized cross-checks against the reference .so --------------------------------------
@needs_ref
def test_restatement_vs_reference_random():
    R = reference()
    rng = np.random.default_rng(5)
    for trial in range(12):
        shapes = [tuple(int(x) for x in rng.integers(1, 90, size=int(rng.integers(1, 4)))) for _ in range(int(rng.integers(1, 4)))]
        sp = float(rng.choice([0.0, 0.5, 0.9, 0.99, 1.0]))
        prev, curr = R.generate_synthetic(shapes, sp, int(rng.integers(1, 40)), trial)
        for r in (0, 1, 2):
            a = R.encode(curr, prev, r, IDENTITY)
            b = S.encode(curr, prev, r, IDENTITY)
            assert R.write_patch_bytes(a) == S.write_patch_bytes_identity(b)


@needs_ref
def test_reference_bf16_rounding_samples():
    R = reference()
    assert R.round_to_bf16(1.0) == 0x3F80
    assert R.round_to_bf16(1.008) == 0x3F81
    assert R.round_to_bf16(float("nan")) == 0x7FC0
