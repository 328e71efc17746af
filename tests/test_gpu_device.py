"""GPU parity of the device-resident path (K1/K2 encode, D* apply) against
the reference's own bytes (golden fixtures + oracle/_ref) on the same inputs."""
import struct

import numpy as np
import pytest

from oracle.oracle import COO_DOWNSCALED, COO_INT32, FLAT_INT32, IDENTITY, have_reference, reference, restatement

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev():
    from paper_2602_03839_b200 import device as D
    return D


def split_pulp(wire: bytes):
    """PULP -> (header dict, body bytes)  (patch_file.hpp:30-83)."""
    import json
    assert wire[:4] == b"PULP"
    ver, hlen = struct.unpack_from("<IQ", wire, 4)
    return json.loads(wire[16:16 + hlen]), wire[16 + hlen:]


def upload(ck):
    ts = ck.sorted()
    return ts, [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in ts]


def make_plan(ts, max_changes=None):
    D = _dev()
    geoms = [(t.data.size, t.shape[-1]) for t in ts]
    cap = max_changes or max(16, sum(t.data.size for t in ts))
    return D.DevicePlan(geoms, cap)


@pytest.fixture(params=["auto", "sparse", "sparse_low", "dense", "dense2", "dense3"])
def k1_shape(request, monkeypatch):
    """K1's staging shape (encode.cu tma::SparseCfg / DenseCfg / Dense2Cfg / Dense3Cfg): chosen from the
    plan's capacity, or forced through PULSE_K1_SHAPE so each runs on every golden case."""
    if request.param != "auto":
        monkeypatch.setenv("PULSE_K1_SHAPE", request.param)
    return request.param


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
def test_encode_body_matches_reference_pulp(golden, repr_, k1_shape):
    for name in golden.names:
        prev, curr, m = golden.case(name)
        want = golden.pulp(name, repr_, IDENTITY)
        if want is None:
            continue
        header, body = split_pulp(want)
        ts, prev_d = upload(prev)
        _, curr_d = upload(curr)
        plan = make_plan(ts)
        plan.bind(0, prev_d)
        plan.bind(1, curr_d)
        p = plan.encode(1, 0, repr_)
        p.raise_for_status([t.name for t in ts])
        assert p.n_entries == len(header["tensors"]), name
        got = p.body[: p.body_bytes].cpu().numpy().tobytes()
        assert got == body, (name, repr_)
        for e, h in zip(p.host_entries, header["tensors"]):
            assert ts[int(e["tensor"])].name == h["name"]
            assert int(e["count"]) == h["count"]
            assert int(e["idx_nbytes"]) == h["index_nbytes"]


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
def test_apply_rebuilds_current_bitwise(golden, repr_):
    for name in golden.names:
        prev, curr, _ = golden.case(name)
        ts, prev_d = upload(prev)
        _, curr_d = upload(curr)
        _, w_d = upload(prev)
        plan = make_plan(ts)
        plan.bind(0, prev_d)
        plan.bind(1, curr_d)
        plan.bind(2, w_d)
        p = plan.encode(1, 0, repr_)
        res = _dev().parse_result(plan.apply(2, p))
        assert int(res["status"]) == 0, (name, res)
        for a, b in zip(w_d, curr_d):
            assert torch.equal(a, b), name
        # decode-only path returns the reference's indices
        idx, res = plan.decode_indices(p)
        ref_idx = np.concatenate([restatement().diff(q.data, c.data)[0] for q, c in zip(prev.sorted(), curr.sorted())])
        assert np.array_equal(idx.cpu().numpy(), ref_idx), name


def test_empty_patch_and_identical_snapshots():
    D = _dev()
    x = torch.arange(4096, dtype=torch.int16, device="cuda")
    plan = D.DevicePlan([(4096, 64)], 100)
    plan.bind(0, [x])
    plan.bind(1, [x.clone()])
    for r in (0, 1, 2):
        p = plan.encode(1, 0, r)
        assert p.status == 0 and p.n_entries == 0 and p.body_bytes == 0 and p.n_changes == 0


def test_capacity_overflow_is_reported():
    D = _dev()
    a = torch.zeros(10000, dtype=torch.int16, device="cuda")
    b = torch.ones(10000, dtype=torch.int16, device="cuda")
    plan = D.DevicePlan([(10000, 100)], 100)
    plan.bind(0, [a])
    plan.bind(1, [b])
    p = plan.encode(1, 0, COO_INT32)
    assert p.status == 15 and int(p.host_result["required"]) == 10000


def test_large_tensor_tiles_and_partial_tail():
    """Several tensors, sizes not multiples of the 8192-element tile, dense and sparse regions."""
    D = _dev()
    R = restatement()
    rng = np.random.default_rng(3)
    sizes = [(8192 * 3 + 40, 8), (17, 17), (8192, 4096), (1000008, 24)]
    prevs, currs = [], []
    for n, _ in sizes:
        a = rng.integers(0, 65536, n, dtype=np.uint16)
        b = a.copy()
        k = rng.random(n) < rng.choice([0.001, 0.01, 0.5])
        b[k] ^= 1
        prevs.append(a)
        currs.append(b)
    plan = D.DevicePlan(sizes, sum(n for n, _ in sizes))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
    for repr_ in (0, 1, 2):
        p = plan.encode(1, 0, repr_)
        assert p.status == 0
        idx, _ = plan.decode_indices(p)
        want = np.concatenate([R.diff(a, b)[0] for a, b in zip(prevs, currs)])
        assert np.array_equal(idx.cpu().numpy(), want)


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
def test_config1_16m_matches_reference_bytes(golden):
    """BASELINE configs[0]: 4096^2, 99%, cluster 64, seed 7 from the reference
    generator itself; the device body must equal the reference PULP body."""
    R = reference()
    prev, curr = R.generate_synthetic([(4096, 4096)], 0.99, 64, 7)
    ts, prev_d = upload(prev)
    _, curr_d = upload(curr)
    plan = make_plan(ts, 400000)
    plan.bind(0, prev_d)
    plan.bind(1, curr_d)
    for r in (0, 1, 2):
        p = plan.encode(1, 0, r)
        assert p.n_changes == golden.manifest["config1"]["changes"] == 167772
        want = R.write_patch_bytes(R.encode(curr, prev, r, IDENTITY))
        header, body = split_pulp(want)
        assert p.body[: p.body_bytes].cpu().numpy().tobytes() == body
        assert len(want) == golden.manifest["config1"]["pulp_nbytes"][f"{r}/0"]


@pytest.mark.parametrize("shape", ["sparse", "sparse_low", "dense", "dense2", "dense3"])
def test_dense_ticket_slow_path(shape, monkeypatch):
    monkeypatch.setenv("PULSE_K1_SHAPE", shape)
    _dense_ticket_slow_path()


def _dense_ticket_slow_path():
    """A fully changed ticket overflows the shared-memory staging of K1 and is
    re-streamed from global memory; results must not change."""
    D = _dev()
    R = restatement()
    n = 65536 * 3 + 1000
    a = np.arange(n, dtype=np.uint16)
    b = a ^ 1
    b[70000:80000] = a[70000:80000]  # one sparse region in the middle
    plan = D.DevicePlan([(n, 8)], n)
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda()])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda()])
    for repr_ in (0, 1, 2):
        p = plan.encode(1, 0, repr_)
        assert p.status == 0 and p.n_changes == n - 10000
        idx, _ = plan.decode_indices(p)
        assert np.array_equal(idx.cpu().numpy(), R.diff(a, b)[0])


def _corrupt_last_entry(p, repr_, ts):
    """Corrupt the final index entry of the last changed tensor in place while
    keeping the fixed (escape-free) layout: a column past the row for
    COO_DOWNSCALED, a gap far past the tensor for the int32 representations."""
    e = p.host_entries[p.n_entries - 1]
    body = p.body
    off, cnt = int(e["idx_off"]), int(e["count"])
    if repr_ == COO_DOWNSCALED:
        pos = off + cnt + 2 * (cnt - 1)           # last column unit
        body[pos] = 0xFE
        body[pos + 1] = 0xFF                      # 0xFFFE: not a marker, > any column extent used here
    else:
        pos = off + 4 * (cnt - 1)                 # last u32 gap
        body[pos:pos + 4] = torch.tensor([0xF0, 0xFF, 0xFF, 0x7F], dtype=torch.uint8, device=body.device)
    return pos


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
def test_corrupt_patch_never_half_applies(repr_):
    """A late bad entry: apply reports the reference's error kind and the
    weights are bit-identical to before (checked writes + restore)."""
    D = _dev()
    R = restatement()
    rng = np.random.default_rng(11)
    sizes = [(300 * 1000, 1000), (70000, 700), (4096 * 64, 4096)]
    prevs = [rng.integers(0, 65536, n, dtype=np.uint16) for n, _ in sizes]
    currs = []
    for a in prevs:
        b = a.copy()
        b[rng.random(a.size) < 0.02] ^= 1
        currs.append(b)
    plan = D.DevicePlan(sizes, sum(n for n, _ in sizes))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
    w = [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs]
    plan.bind(2, w)
    p = plan.encode(1, 0, repr_)
    assert p.status == 0
    _corrupt_last_entry(p, repr_, sizes)
    res = D.parse_result(plan.apply(2, p))
    assert int(res["status"]) in (7, 11), res          # CorruptStreamError (reference kind for these)
    assert int(res["status"]) == 7
    for a, t in zip(prevs, w):
        assert np.array_equal(t.cpu().numpy().view(np.uint16), a)   # nothing half-applied
    # and a clean patch still applies after the failed one
    p2 = plan.encode(1, 0, repr_)
    assert int(D.parse_result(plan.apply(2, p2))["status"]) == 0
    for b, t in zip(currs, w):
        assert np.array_equal(t.cpu().numpy().view(np.uint16), b)


def test_apply_rejects_more_entries_than_capacity():
    D = _dev()
    n = 50000
    a = np.arange(n, dtype=np.uint16)
    b = a ^ 1
    big = D.DevicePlan([(n, 100)], n)
    big.bind(0, [torch.from_numpy(a.view(np.int16)).cuda()])
    big.bind(1, [torch.from_numpy(b.view(np.int16)).cuda()])
    p = big.encode(1, 0, COO_DOWNSCALED)
    small = D.DevicePlan([(n, 100)], 1000)
    w = torch.from_numpy(a.view(np.int16)).cuda()
    small.bind(2, [w])
    res = D.parse_result(small.apply(2, p))
    assert int(res["status"]) == 15
    assert np.array_equal(w.cpu().numpy().view(np.uint16), a)


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
def test_apply_patch_device_count_and_failed_encode(repr_):
    """pulse_apply_patch takes the entry count from the encode's device result;
    a failed encode (capacity) applies nothing and reports the encode's error."""
    D = _dev()
    rng = np.random.default_rng(5)
    sizes = [(40000, 200), (12345, 5), (9000, 9000)]
    prevs = [rng.integers(0, 65536, n, dtype=np.uint16) for n, _ in sizes]
    currs = []
    for a in prevs:
        b = a.copy()
        b[rng.random(a.size) < 0.05] ^= 1
        currs.append(b)
    for cap, ok in ((sum(n for n, _ in sizes), True), (100, False)):
        plan = D.DevicePlan(sizes, cap)
        plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
        plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
        w = [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs]
        plan.bind(2, w)
        p = plan.new_patch(repr_)
        plan.scan(1, 0)
        plan.emit(p)
        res = D.parse_result(plan.apply_patch(2, p))   # no host fetch in between
        if ok:
            assert int(res["status"]) == 0
            for b, t in zip(currs, w):
                assert np.array_equal(t.cpu().numpy().view(np.uint16), b)
        else:
            assert int(res["status"]) == 15
            for a, t in zip(prevs, w):
                assert np.array_equal(t.cpu().numpy().view(np.uint16), a)


@pytest.mark.parametrize("numel,cols", [((1 << 31) + (1 << 20) + 24, 4096 + 8), ((1 << 32) + 4096, 1 << 20)])
def test_segmented_and_wide_tensors_round_trip(numel, cols):
    """Tensors past 2^31 elements are split into 32-bit segments by K1/K2; past
    2^32 the index coding and apply take their 64-bit paths.  Size-independent
    checks: exact change count, exact round trip for every representation, and
    the decoded indices around the segment boundary against a host diff."""
    D = _dev()
    if torch.cuda.get_device_properties(0).total_memory < 60 * (1 << 30):
        pytest.skip("needs a large-memory GPU")
    rows = numel // cols
    n = rows * cols
    prev = torch.empty(n, dtype=torch.int16, device="cuda")
    curr = torch.empty_like(prev)
    D.synth_base(prev, seed=5)
    changed = D.synth_mutate(prev, curr, 0.9999, 64, seed=6)
    # force changes right around the 2^31 split and the last element
    for p in [(1 << 31) - 2, (1 << 31) - 1, 1 << 31, (1 << 31) + 1, n - 1]:
        if p < n:
            curr[p] = prev[p] ^ 1
    torch.cuda.synchronize()
    want = int((curr != prev).sum().item())
    plan = D.DevicePlan([(n, cols)], want + 1024)
    w = prev.clone()
    plan.bind(0, [prev])
    plan.bind(1, [curr])
    plan.bind(2, [w])
    for repr_ in (COO_DOWNSCALED, COO_INT32, FLAT_INT32):
        p = plan.encode(1, 0, repr_)
        if repr_ != COO_DOWNSCALED and n >= (1 << 31):
            assert p.status == 12  # DimensionError: int32 representations reject 2^31+ tensors (patch.hpp:99-103)
            continue
        assert p.status == 0 and p.n_changes == want, (repr_, p.status)
        idx, _ = plan.decode_indices(p)
        lo, hi = (1 << 31) - 4096, (1 << 31) + 4096
        seg = idx[(idx >= lo) & (idx < hi)].cpu().numpy()
        ref = (torch.nonzero(curr[lo:hi] != prev[lo:hi]).flatten() + lo).cpu().numpy()
        assert np.array_equal(seg, ref)
        w.copy_(prev)
        res = D.parse_result(plan.apply(2, p))
        assert int(res["status"]) == 0
        assert torch.equal(w, curr)
    del prev, curr, w
    torch.cuda.empty_cache()


def _first_failure(repr_, entries, body, sizes, has_prev=False):
    """The reference's first failing (entry, check, ordinal) for a fixed-layout body
    (patch.hpp:178-262, index_coding.hpp:130-158), or None; numpy restatement used
    as the checker for the corruption tests below."""
    glob = 0
    any_decoded = has_prev
    flat_base = 0
    for k, e in enumerate(entries):
        t = int(e["tensor"])
        numel, cols = sizes[t]
        cnt, off = int(e["count"]), int(e["idx_off"])
        if repr_ == COO_DOWNSCALED:
            rg = np.frombuffer(body, np.uint8, cnt, off).astype(np.int64)
            cv = np.frombuffer(body, "<u2", cnt, off + cnt).astype(np.int64)
            head = rg != 0
            head[0] = True
            zero = np.flatnonzero(~head & (cv == 0))
            if zero.size:
                return k, 3, int(zero[0])
            rows = np.cumsum(rg)
            seg = np.cumsum(head) - 1
            starts = np.flatnonzero(head)
            csum = np.cumsum(cv)
            base = (csum - cv)[starts]
            colv = csum - base[seg]
            bad_c = colv >= cols
            bad_i = rows * cols + colv >= numel
            i = np.flatnonzero(bad_c | bad_i)
            if i.size:
                return k, (4 if bad_c[i[0]] else 5), int(i[0])
        else:
            g = np.frombuffer(body, "<u4", cnt, off).astype(np.int64)
            if repr_ == COO_INT32:
                idx = np.cumsum(g)
                zero = g == 0
                zero[0] = False
                rng_ = idx >= numel
            else:
                gl = glob + np.cumsum(g) if any_decoded else g[0] + np.concatenate([[0], np.cumsum(g[1:])])
                zero = g == 0
                if not any_decoded:
                    zero[0] = False
                local = gl - flat_base
                rng_ = (local < 0) | (local >= numel)
                glob = int(gl[-1])
                any_decoded = True
            i = np.flatnonzero(zero | rng_)
            if i.size:
                return k, (2 if zero[i[0]] else 5), int(i[0])
        flat_base += numel
    return None


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
@pytest.mark.parametrize("where", ["range_start", "slack", "mid_range", "row_jump", "zero_gap"])
def test_mid_tensor_corruption_reports_first_failure(repr_, where):
    """Bad entries deep inside a large tensor (ranges holding no tensor start or
    end, where apply checks without the carry): the first failing entry and
    check are the reference's, and nothing is written."""
    D = _dev()
    rng = np.random.default_rng(5)
    sizes = [(2000 * 4096, 4096), (300 * 700, 700)]
    prevs = [rng.integers(0, 65536, n, dtype=np.uint16) for n, _ in sizes]
    currs = []
    for a in prevs:
        b = a.copy()
        b[rng.random(a.size) < 0.02] ^= 1
        currs.append(b)
    plan = D.DevicePlan(sizes, sum(n for n, _ in sizes))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
    w = [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs]
    plan.bind(2, w)
    p = plan.encode(1, 0, repr_)
    assert p.status == 0
    e0 = p.host_entries[0]
    off, cnt = int(e0["idx_off"]), int(e0["count"])
    assert cnt > 5 * 4096
    body = p.body[: p.body_bytes].cpu().numpy().copy()
    k = 2 * 4096 + (0 if where == "range_start" else 1500)  # entry ordinal in tensor 0 (entries start at 0)
    if repr_ == COO_DOWNSCALED:
        rows = body[off:off + cnt]
        cpos = off + cnt + 2 * k
        if where == "row_jump":
            rows[k:k + 20] = 200                       # rows past the tensor from here on
        elif where == "zero_gap":
            j = k + int(np.flatnonzero(rows[k:] == 0)[0])  # a non-head entry
            cpos = off + cnt + 2 * j
            body[cpos:cpos + 2] = 0
        elif where == "slack":
            # the range's first row segment [r, h) ends exactly at column `cols` while its
            # range-local sum stays below it: only the carry from earlier ranges shows it
            cv = body[off + cnt:off + 3 * cnt].view("<u2").astype(np.int64)
            r = next(x for x in range(k, cnt, 4096) if rows[x] == 0 and rows[x - 1] == 0 and cv[x - 1] > 0)
            h = r + int(np.flatnonzero(rows[r:] != 0)[0])
            hh = r - 1 - int(np.flatnonzero(rows[:r][::-1] != 0)[0])  # head of the row holding r - 1
            carry = int(cv[hh:r].sum())
            local = int(cv[r:h].sum())
            delta = 4096 - carry - local
            assert 0 < carry and 0 < delta and cv[h - 1] + delta < 0xFFFF and local + delta < 4096
            cv[h - 1] += delta
            body[off + cnt:off + 3 * cnt] = cv.astype("<u2").view(np.uint8)
        else:
            j = k + int(np.flatnonzero(rows[k:] == 0)[0])  # a column inside a row
            cpos = off + cnt + 2 * j
            body[cpos:cpos + 2] = [0xFE, 0xFF]
    else:
        pos = off + 4 * k
        if where == "zero_gap":
            body[pos:pos + 4] = 0
        elif where == "row_jump":
            body[pos:pos + 4] = [0, 0, 0, 0x10]       # a 2^28 gap: every later index out of range
        else:
            body[pos:pos + 4] = [0xF0, 0xFF, 0xFF, 0x7F]
    want = _first_failure(repr_, p.host_entries[: p.n_entries], body.tobytes(), sizes)
    assert want is not None
    p.body[: p.body_bytes] = torch.from_numpy(body).cuda()
    res = D.parse_result(plan.apply(2, p))
    assert int(res["status"]) == 7, res
    assert (int(res["err_tensor"]), int(res["err_check"]), int(res["err_elem"])) == want, (res, want)
    for a, t in zip(prevs, w):
        assert np.array_equal(t.cpu().numpy().view(np.uint16), a)


def test_clean_patch_checks_pass_on_plain_ranges():
    """No false alarm: a large clean patch in every representation applies exactly
    (the carry-free checks of plain ranges and the deferred column check)."""
    D = _dev()
    rng = np.random.default_rng(9)
    sizes = [(3000 * 4096, 4096), (1 << 20, 1 << 20), (1000 * 9, 9)]
    prevs = [rng.integers(0, 65536, n, dtype=np.uint16) for n, _ in sizes]
    currs = []
    for i, a in enumerate(prevs):
        b = a.copy()
        b[rng.random(a.size) < (0.3 if i == 2 else 0.01)] ^= 1
        currs.append(b)
    plan = D.DevicePlan(sizes, sum(n for n, _ in sizes))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
    for repr_ in (COO_DOWNSCALED, COO_INT32, FLAT_INT32):
        w = [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs]
        plan.bind(2, w)
        p = plan.encode(1, 0, repr_)
        res = D.parse_result(plan.apply(2, p))
        assert int(res["status"]) == 0, (repr_, res)
        for b, t in zip(currs, w):
            assert np.array_equal(t.cpu().numpy().view(np.uint16), b)


@pytest.mark.parametrize("case", ["esc_cols", "esc_rows", "handcrafted", "roundtrip_s0"])
@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, FLAT_INT32])
def test_graph_replay_runs_gated_paths(golden, case, repr_):
    """encode + apply captured as a CUDA graph (the benchmark's launch mode): K2's
    exact re-run and the escape-aware decoder sit behind conditional graph nodes.
    Replays in both directions land exactly on the targets and produce the
    reference's body, for patches that need those paths (escapes) and ones that do not."""
    D = _dev()
    prev, curr, m = golden.case(case)
    ts, prev_d = upload(prev)
    _, curr_d = upload(curr)
    plan = make_plan(ts)
    plan.bind(0, prev_d)
    plan.bind(1, curr_d)
    w = [t.clone() for t in prev_d]
    plan.bind(2, w)
    patches = [plan.new_patch(repr_), plan.new_patch(repr_)]
    res = [torch.zeros(72, dtype=torch.uint8, device="cuda") for _ in range(2)]
    stream = torch.cuda.Stream()
    graphs = []
    with torch.cuda.stream(stream):
        for k, (cs, ps) in enumerate(((1, 0), (0, 1))):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                plan.scan(cs, ps, stream=stream)
                plan.emit(patches[k], stream=stream)
                plan.apply_patch(2, patches[k], result=res[k], stream=stream)
            graphs.append(g)
    want = golden.pulp(case, repr_, IDENTITY)
    for rep in range(2):
        for k, target in ((0, curr_d), (1, prev_d)):
            graphs[k].replay()
            torch.cuda.synchronize()
            r = D.parse_result(res[k])
            assert int(r["status"]) == 0, (case, repr_, r)
            for a, b in zip(w, target):
                assert torch.equal(a, b), (case, repr_, rep, k)
            if k == 0 and want is not None:
                patches[0].fetch()
                _, body = split_pulp(want)
                assert patches[0].body[: patches[0].body_bytes].cpu().numpy().tobytes() == body


@pytest.mark.parametrize("repr_", [COO_DOWNSCALED, COO_INT32, FLAT_INT32])
def test_many_tiny_tensors_small_plan(repr_):
    """Hundreds of tiny tensors under a plan sized for few changes: the list of
    pieces F3 checks overflows, apply falls back to exact checks of every range,
    and both a clean and a corrupted patch behave exactly as the reference's."""
    D = _dev()
    rng = np.random.default_rng(17)
    sizes = [(int(rng.integers(1, 50)) * 64, 64) for _ in range(700)]  # row gaps < 255: no escapes
    prevs = [rng.integers(0, 65536, n, dtype=np.uint16) for n, _ in sizes]
    currs = []
    for a in prevs:
        b = a.copy()
        b[rng.integers(0, a.size, 2)] ^= 1
        currs.append(b)
    total_changes = sum(int((a != b).sum()) for a, b in zip(prevs, currs))
    plan = D.DevicePlan(sizes, max(1024, total_changes))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs])
    plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda() for b in currs])
    w = [torch.from_numpy(a.view(np.int16)).cuda() for a in prevs]
    plan.bind(2, w)
    p = plan.encode(1, 0, repr_)
    assert p.status == 0 and p.n_changes == total_changes
    body = p.body[: p.body_bytes].cpu().numpy().copy()
    res = D.parse_result(plan.apply(2, p))
    assert int(res["status"]) == 0, res
    for b, t in zip(currs, w):
        assert np.array_equal(t.cpu().numpy().view(np.uint16), b)
    # corrupt one entry in the middle tensor: the reference's first failure, nothing written
    for a, t in zip(prevs, w):
        t.copy_(torch.from_numpy(a.view(np.int16)))
    e = p.host_entries[p.n_entries // 2]
    off, cnt = int(e["idx_off"]), int(e["count"])
    if repr_ == COO_DOWNSCALED:
        body[off + cnt:off + cnt + 2] = [0xFE, 0xFF]   # first column entry past any row
    else:
        body[off:off + 4] = [0xF0, 0xFF, 0xFF, 0x7F]
    want = _first_failure(repr_, p.host_entries[: p.n_entries], body.tobytes(), sizes)
    p.body[: p.body_bytes] = torch.from_numpy(body).cuda()
    res = D.parse_result(plan.apply(2, p))
    assert int(res["status"]) == 7
    assert (int(res["err_tensor"]), int(res["err_check"]), int(res["err_elem"])) == want
    for a, t in zip(prevs, w):
        assert np.array_equal(t.cpu().numpy().view(np.uint16), a)


# ---- out-of-bounds writes: canaries around every caller buffer -----------------------------------
# (compute-sanitizer is not available on the GPU pool; these guard bytes catch a kernel that writes
# past a weight tensor, the patch body, the entry table or the result record)
_CANARY = 0x5A


def _guarded(n, dtype, pad):
    """A view of n elements inside a buffer of canary bytes (pad elements each side, 16-byte aligned)."""
    base = torch.full((n + 2 * pad,), 0, dtype=dtype, device="cuda")
    base.view(torch.uint8).fill_(_CANARY)
    return base, base[pad:pad + n]


def _intact(base, view, pad):
    b = base.view(torch.uint8).cpu().numpy()
    es = base.element_size()
    return bool((b[: pad * es] == _CANARY).all() and (b[(pad + view.numel()) * es:] == _CANARY).all())


@pytest.mark.parametrize("case", ["handcrafted", "esc_rows", "esc_cols", "esc_cols_wide", "dense_all",
                                  "h5_unchanged", "h5_sparse_lead", "roundtrip_s3"])
def test_no_writes_outside_caller_buffers(golden, case, k1_shape):
    D = _dev()
    prev, curr, _ = golden.case(case)
    ts = prev.sorted()
    cs = curr.sorted()
    PAD = 4096
    # weights: each tensor between canaries
    wbufs = [_guarded(t.data.size, torch.int16, PAD) for t in ts]
    pd = [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in ts]
    cd = [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in cs]
    plan = make_plan(ts)
    plan.bind(0, pd)
    plan.bind(1, cd)
    plan.bind(2, [v for _, v in wbufs])
    for r in (COO_DOWNSCALED, COO_INT32, FLAT_INT32):
        want = golden.pulp(case, r, IDENTITY)
        _, body = split_pulp(want)
        for cap in (len(body), max(0, len(body) - 1), len(body) // 2, 16, plan.body_capacity(r)):
            bb, bv = _guarded(max(cap, 1), torch.uint8, PAD)
            eb, ev = _guarded(max(1, len(ts)) * 40, torch.uint8, PAD)
            rb, rv = _guarded(72, torch.uint8, PAD)
            p = D.DevicePatch(r, bv[:cap] if cap else bv[:0], ev, rv)
            plan.scan(1, 0)
            plan.emit(p)
            p.fetch()
            assert _intact(bb, bv, PAD) and _intact(eb, ev, PAD) and _intact(rb, rv, PAD), (case, r, cap)
            if cap >= len(body):
                assert p.status == 0 and p.body[: p.body_bytes].cpu().numpy().tobytes() == body
                for (wb, wv), a in zip(wbufs, pd):
                    wv.copy_(a)
                res = D.parse_result(plan.apply(2, p))
                assert int(res["status"]) == 0
                assert all(torch.equal(wv, c) for (_, wv), c in zip(wbufs, cd))
                assert all(_intact(wb, wv, PAD) for wb, wv in wbufs), (case, r)
                idx, _ = plan.decode_indices(p)
            else:
                assert p.status == 15 and int(p.host_result["required"]) >= len(body), (case, r, cap, p.status)
