"""The Python mirror of the reference API (paper_2602_03839_b200.host) over the
host-buffer C ABI, against the reference's own bytes: full PULP files (every
representation x codec) from encode -> write_patch_bytes, read -> decode
round trips, index payload coding, and the host-only helpers (hash, codecs)."""
import numpy as np
import pytest

from oracle.oracle import have_reference, reference

H = pytest.importorskip("paper_2602_03839_b200.host")

CODECS = [0, 1, 2, 3, 4]


def mirror(ck):
    return H.Checkpoint(ck.step, [H.Tensor(t.name, t.shape, t.data) for t in ck.tensors])


def as_ref_patch(p):
    from oracle.oracle import Patch, TensorPatch
    return Patch(p.base_step, p.target_step, p.anchor_step, p.representation, p.codec, p.target_hash,
                 [TensorPatch(t.name, t.shape, t.indices, t.values) for t in p.tensors])


# ---- host-only (CPU) --------------------------------------------------------------------------
def test_hash_weights_matches_golden(golden):
    for name in golden.names:
        _, curr, m = golden.case(name)
        assert H.hash_weights(mirror(curr)).hex() == m["target_hash"], name


@pytest.mark.parametrize("codec", CODECS)
def test_codec_round_trip_and_bytes(codec):
    rng = np.random.default_rng(codec)
    data = (rng.integers(0, 4, 200_000, dtype=np.uint8)).tobytes()
    z = H.compress(data, codec)
    assert H.decompress(z, codec) == data
    if have_reference():
        assert z == reference().compress(data, codec)


def test_transfer_stats_exported():
    h2d, d2h = H.transfer_stats()
    assert h2d >= 0 and d2h >= 0


# ---- device compute through the host API --------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("repr_", [0, 1, 2])
def test_encode_write_matches_reference_pulp(golden, repr_):
    for name in golden.names:
        prev, curr, m = golden.case(name)
        for codec in CODECS:
            want = golden.pulp(name, repr_, codec)
            if want is None:
                continue
            h = H.encode_handle(mirror(curr), mirror(prev), repr_, codec)
            assert H.write_patch_bytes(h) == want, (name, repr_, codec)
            arr = H.write_patch_array(h)
            assert arr.tobytes() == want
            assert H.read_patch_handle(arr).to_patch().total_changes() == H.read_patch_bytes(want).total_changes()


@pytest.mark.gpu
@pytest.mark.parametrize("repr_", [0, 1, 2])
def test_read_decode_round_trip(golden, repr_):
    for name in golden.names:
        prev, curr, m = golden.case(name)
        for codec in CODECS:
            wire = golden.pulp(name, repr_, codec)
            if wire is None:
                continue
            p = H.read_patch_bytes(wire)
            assert p.total_changes() == m["patches"][f"{repr_}/{codec}"]["changes"]
            out = H.decode(mirror(prev), p, verify_hash=True)
            for a, b in zip(sorted(out.tensors, key=lambda t: t.name), curr.sorted()):
                assert np.array_equal(a.data, b.data), (name, repr_, codec, a.name)


@pytest.mark.gpu
def test_patch_object_matches_reference_encode(golden):
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = reference()
    for name in golden.names[:6]:
        prev, curr, _ = golden.case(name)
        for repr_ in (0, 1, 2):
            mine = H.encode(mirror(curr), mirror(prev), repr_, 2)
            ref = R.encode(curr, prev, repr_, 2)
            assert mine.target_hash == ref.target_hash
            assert [t.name for t in mine.tensors] == [t.name for t in ref.tensors]
            for a, b in zip(mine.tensors, ref.tensors):
                assert np.array_equal(a.indices, b.indices) and np.array_equal(a.values, b.values)
            pay = H.encode_index_payloads(mine)
            assert pay == R.encode_index_payloads(ref), (name, repr_)
            back = H.decode_index_payloads(H.SparsePatch(mine.base_step, mine.target_step, mine.anchor_step,
                                                         repr_, 2, mine.target_hash,
                                                         [H.TensorPatch(t.name, t.shape, np.zeros(0, np.int64),
                                                                        t.values) for t in mine.tensors]), pay)
            for a, b in zip(back.tensors, mine.tensors):
                assert np.array_equal(a.indices, b.indices)


@pytest.mark.gpu
def test_index_helpers_match_reference():
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = reference()
    rng = np.random.default_rng(3)
    idx = np.unique(rng.integers(0, 1 << 40, 50_000)).astype(np.int64)
    g = H.delta_encode_indices(idx)
    assert np.array_equal(g, R.delta_encode(idx))
    assert np.array_equal(H.delta_decode_indices(g), idx)
    rows = np.sort(rng.integers(0, 1 << 20, 20_000)).astype(np.int64)
    cols = rng.integers(0, 1 << 18, 20_000).astype(np.int64)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.concatenate([[True], (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])])
    rows, cols = rows[keep], cols[keep]
    b = H.downscale_coo(rows, cols)
    assert b == R.downscale_coo(rows, cols)
    r2, c2 = H.upscale_coo(b, rows.size)
    assert np.array_equal(r2, rows) and np.array_equal(c2, cols)


@pytest.mark.gpu
def test_errors_map_to_reference_kinds(golden):
    from oracle.oracle import OracleError, Tensor

    prev, curr, _ = golden.case("roundtrip_s0")
    R = reference() if have_reference() else None
    for codec in CODECS:
        wire = golden.pulp("roundtrip_s0", 0, codec)
        for cut in (3, 40, len(wire) - 10):
            with pytest.raises(H.PulseError) as e:
                H.read_patch_bytes(wire[:-cut])
            if R is not None:
                with pytest.raises(OracleError) as r:
                    R.read_patch_bytes(wire[:-cut])
                assert e.value.kind == r.value.kind, (codec, cut)
    wire = golden.pulp("roundtrip_s0", 0, 2)
    bad = mirror(prev)
    bad.tensors[0] = H.Tensor(bad.tensors[0].name, (1,), bad.tensors[0].data[:1])
    with pytest.raises(H.PulseError) as e:
        H.decode(bad, H.read_patch_bytes(wire))
    if R is not None:
        rb = type(prev)(prev.step, [Tensor(t.name, t.shape, t.data) for t in bad.tensors])
        with pytest.raises(OracleError) as r:
            R.decode(rb, R.read_patch_bytes(wire))
        assert e.value.kind == r.value.kind


# ---- absorption.hpp analyses (row a21 + frozen_fraction) ------------------------------------------
@pytest.mark.gpu
def test_sparsity_matches_reference(golden):
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = reference()
    for name in golden.names:
        prev, curr, m = golden.case(name)
        r = H.sparsity(mirror(curr), mirror(prev), k=3)
        ch, tot = R.sparsity(curr, prev)
        assert (r.changed, r.total, r.k) == (ch, tot, 3), name
        assert r.sparsity == (1.0 - ch / tot if tot else 1.0)
        assert H.sparsity(mirror(prev), mirror(prev)).changed == 0


@pytest.mark.gpu
def test_frozen_fraction_matches_reference_and_numpy(golden):
    rng = np.random.default_rng(9)
    bits = rng.integers(0, 65536, 300001, dtype=np.uint16)
    bits[:8] = [0x0000, 0x8000, 0x7F80, 0xFF80, 0x7FC0, 0xFFC1, 0x0001, 0x3F80]  # zeros, infs, NaNs, subnormal, 1.0
    c = H.Checkpoint(0, [H.Tensor("w", (300001,), bits)])
    with np.errstate(invalid="ignore"):  # NaN patterns
        f32 = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    for t in [0.0, 1.0, 0.25, 7.68e-4, 1e-40, -1.0, float("inf"), float("nan"), 3.0e38, 2.0 ** -133]:
        want = float(np.count_nonzero(np.abs(f32) > t)) / bits.size
        got = H.frozen_fraction(c, t)
        assert got == want, (t, got, want)
        if have_reference():
            from oracle.oracle import Checkpoint, Tensor
            assert got == reference().frozen_fraction(Checkpoint(0, [Tensor("w", (300001,), bits)]), t), t
    with pytest.raises(H.PulseError):
        H.frozen_fraction(H.Checkpoint(0, []), 0.1)


@pytest.mark.gpu
def test_sparsity_errors_match_reference():
    a = H.Checkpoint(0, [H.Tensor("w", (2,), np.zeros(2, np.uint16))])
    with pytest.raises(H.PulseError) as e:
        H.sparsity(a, H.Checkpoint(0, [H.Tensor("x", (2,), np.zeros(2, np.uint16))]))
    assert e.value.kind == "TensorSetError"
    with pytest.raises(H.PulseError) as e:
        H.sparsity(a, H.Checkpoint(0, []))
    assert e.value.kind == "TensorSetError"
    with pytest.raises(H.PulseError) as e:
        H.sparsity(a, H.Checkpoint(0, [H.Tensor("w", (2, 1), np.zeros(2, np.uint16))]))
    assert e.value.kind == "ShapeMismatchError"


@pytest.mark.gpu
@pytest.mark.parametrize("repr_", [0, 2])
def test_decode_pipeline_with_pinned_buffers(golden, repr_):
    """Page-locked base and output buffers take the validate-then-pipelined
    (upload | scatter | download) decode; results equal the reference target,
    and a failing decode leaves the outputs untouched."""
    torch = pytest.importorskip("torch")
    for name in ("roundtrip_s1", "esc_rows", "handcrafted"):
        prev, curr, _ = golden.case(name)
        pins = [torch.from_numpy(t.data.view(np.int16).copy()).pin_memory() for t in prev.tensors]
        outs = [torch.empty_like(p).pin_memory() for p in pins]
        pc = H.Checkpoint(prev.step, [H.Tensor(t.name, t.shape, p.numpy().view(np.uint16))
                                      for t, p in zip(prev.tensors, pins)])
        h = H.encode_handle(mirror(curr), mirror(prev), repr_, 0)
        back = H.read_patch_handle(H.write_patch_array(h))
        H.decode_into(pc, back, [o.numpy().view(np.uint16) for o in outs], verify_hash=True)
        want = {t.name: t.data for t in curr.tensors}
        for t, o in zip(prev.tensors, outs):
            assert np.array_equal(o.numpy().view(np.uint16), want[t.name]), (name, t.name)
        # corrupt: a patch whose shape no longer fits -> error, outputs unchanged
        sentinel = [o.clone() for o in outs]
        bad = H.read_patch_handle(H.write_patch_array(h)).to_patch()
        if bad.tensors:
            t0 = bad.tensors[0]
            bad.tensors[0] = H.TensorPatch(t0.name, t0.shape, t0.indices.copy(), t0.values)
            bad.tensors[0].indices[-1] = np.prod(t0.shape) + 5   # past the tensor
            with pytest.raises(H.PulseError):
                H.decode_into(pc, H.PatchHandle.from_patch(bad), [o.numpy().view(np.uint16) for o in outs],
                              verify_hash=False)
            for o, s_ in zip(outs, sentinel):
                assert torch.equal(o, s_)


@pytest.mark.gpu
def test_host_api_on_two_devices_in_one_process(golden):
    """Launch configuration (shared-memory opt-in, occupancy) is per device: one
    process driving two GPUs round-trips on both."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    prev, curr, _ = golden.case("esc_rows")
    for dev in (0, 1, 0):
        torch.cuda.set_device(dev)
        for repr_ in (0, 1, 2):
            h = H.encode_handle(mirror(curr), mirror(prev), repr_, 2)
            out = H.decode(mirror(prev), H.read_patch_handle(H.write_patch_array(h)), verify_hash=True)
            for a, b in zip(sorted(out.tensors, key=lambda t: t.name), curr.sorted()):
                assert np.array_equal(a.data, b.data), (dev, repr_)
    torch.cuda.set_device(0)


@pytest.mark.gpu
def test_index_helpers_large_and_errors_match_reference():
    """delta_decode_indices / downscale_coo at sizes spanning many scan blocks, the first
    failure deep inside, and downscale_coo entries that all take both escapes (11 bytes
    each) right after a small call sized the library's scratch (the advisor's overrun case)."""
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    from oracle.oracle import OracleError
    R = reference()
    rng = np.random.default_rng(11)
    gaps = rng.integers(1, 1000, 3_000_000).astype(np.int64)
    idx = np.cumsum(gaps)
    assert np.array_equal(H.delta_decode_indices(gaps), idx)
    bad = gaps.copy()
    bad[2_345_678] = 0
    bad[2_900_000] = -5
    with pytest.raises(H.PulseError) as ei:
        H.delta_decode_indices(bad)
    with pytest.raises(OracleError) as er:
        R.delta_decode(bad)
    assert ei.value.kind == er.value.kind
    rows = np.sort(rng.integers(0, 1 << 30, 2_000_000)).astype(np.int64)
    cols = rng.integers(0, 1 << 17, 2_000_000).astype(np.int64)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.concatenate([[True], (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])])
    rows, cols = rows[keep], cols[keep]
    assert H.downscale_coo(rows, cols) == R.downscale_coo(rows, cols)
    # small call first, then entries that all need the row and the column escape
    H.downscale_coo(np.array([0, 1], np.int64), np.array([0, 0], np.int64))
    m = 200_000
    r2 = (np.arange(m, dtype=np.int64) + 1) * 300    # row gaps (and the first row) 300 >= 255
    c2 = np.full(m, 70_000, dtype=np.int64)          # every entry a new row, column 70000 >= 65535
    want = R.downscale_coo(r2, c2)
    assert len(want) == 11 * m
    assert H.downscale_coo(r2, c2) == want
    r3, c3 = r2.copy(), c2.copy()
    r3[150_000] = r3[149_999]                        # same row, column not increasing
    with pytest.raises(H.PulseError) as ei:
        H.downscale_coo(r3, c3)
    with pytest.raises(OracleError) as er:
        R.downscale_coo(r3, c3)
    assert ei.value.kind == er.value.kind and str(ei.value).endswith(er.value.msg)


@pytest.mark.gpu
def test_upscale_coo_parallel_matches_reference():
    """upscale_coo (index_coding.hpp:130-158) on the general decoder's parallel parse:
    large payloads with and without escapes, and damaged ones (truncated row / column
    streams, trailing bytes, zero column gaps, injected 0xFF / 0xFFFF markers) give the
    reference's coordinates or its exception class and message."""
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    from oracle.oracle import OracleError
    R = reference()
    rng = np.random.default_rng(12)
    for n, rmax, cmax in ((1_000_000, 1 << 22, 4000), (300_000, 1 << 31, 1 << 20), (50, 300, 70_000)):
        rows = np.sort(rng.integers(0, rmax, n)).astype(np.int64)
        cols = rng.integers(0, cmax, n).astype(np.int64)
        order = np.lexsort((cols, rows))
        rows, cols = rows[order], cols[order]
        keep = np.concatenate([[True], (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])])
        rows, cols = rows[keep], cols[keep]
        blob = R.downscale_coo(rows, cols)
        r2, c2 = H.upscale_coo(blob, rows.size)
        assert np.array_equal(r2, rows) and np.array_equal(c2, cols)
        variants = [blob[:-1], blob[: len(blob) // 2], blob + b"\x00", blob[:3]]
        for _ in range(30):
            b = bytearray(blob)
            p = int(rng.integers(0, len(b)))
            b[p:p + 2] = rng.choice([b"\xff\xff", b"\x00\x00", b"\xff", b"\x00"])
            variants.append(bytes(b))
        for v in variants:
            try:
                want = ("ok", R.upscale_coo(v, rows.size))
            except OracleError as e:
                want = (e.kind, e.msg)
            try:
                got = ("ok", H.upscale_coo(v, rows.size))
            except H.PulseError as e:
                got = (e.kind, str(e).split(": ", 1)[1])
            assert got[0] == want[0], (got[0], want[0])
            if want[0] == "ok":
                assert np.array_equal(got[1][0], want[1][0]) and np.array_equal(got[1][1], want[1][1])
            else:
                assert got[1] == want[1]
    assert H.upscale_coo(b"", 0)[0].size == 0
