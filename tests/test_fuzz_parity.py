"""Adversarial parity: seeded mutations of the reference's own PULP files.

Every mutated file goes through the reference (oracle/_ref) and through this
library's host API, and both must agree exactly:

* read_patch_bytes (patch_file.hpp:85-147, then decode_index_payloads
  patch.hpp:178-262 / upscale_coo index_coding.hpp:130-158): the same
  exception class AND message, or the same decoded patch (names, shapes,
  indices, values, header fields);
* decode (patch.hpp:309-348, verify_hash=True) of every patch both accept:
  the same exception class and message, or the same weights -- including
  patches with duplicate tensor names (applied in order, last wins) and
  unsorted names, which read_patch_bytes accepts;
* Resident.apply (apply_delta, sync.hpp:308-329) on a sample: the reference's
  error class (read errors first, then decode's), and on failure the held
  weights and step are untouched.

Mutations: bit flips in index / value blobs, injected 0xFF / 0xFFFF marker
runs, zeroed gap bytes, truncation at any offset, count / index_nbytes /
value_nbytes edits with the blobs resized to stay parseable, shape edits,
renamed, duplicated and swapped tensors, and header byte noise.  The failing
mutations are written to gpurun_out/fuzz_mismatches.json for triage.
"""
import json
import os
import struct

import numpy as np
import pytest

from oracle.oracle import OracleError, have_reference, reference

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")]

CASES = ["roundtrip_s0", "roundtrip_s1", "patchfile_s1", "accept_b", "esc_rows", "esc_cols", "esc_cols_wide",
         "handcrafted", "h5_unchanged", "h5_sparse_lead", "dense_all", "accept_c"]
N_MUTATIONS = int(os.environ.get("PULSE_FUZZ_N", "10000"))


def _H():
    from paper_2602_03839_b200 import host
    return host


def _mirror(ck):
    H = _H()
    return H.Checkpoint(ck.step, [H.Tensor(t.name, t.shape, t.data) for t in ck.tensors])


def parse_layout(wire):
    _, hl = struct.unpack_from("<IQ", wire, 4)
    hdr = json.loads(wire[16:16 + hl])
    pos, blobs = 16 + hl, []
    for t in hdr["tensors"]:
        ib = wire[pos:pos + t["index_nbytes"]]
        pos += t["index_nbytes"]
        vb = wire[pos:pos + t["value_nbytes"]]
        pos += t["value_nbytes"]
        blobs.append([ib, vb])
    return hdr, blobs


def assemble(hdr, blobs):
    h = json.dumps(hdr, sort_keys=True, separators=(",", ":")).encode()
    return b"PULP" + struct.pack("<IQ", 1, len(h)) + h + b"".join(i + v for i, v in blobs)


def _guard(pos, codec):
    """Non-identity blobs start with a u64 declared raw size (compression.hpp:
    157-167): bytes 3..7 are left alone so a mutation never declares more than
    16 MiB -- the reference would zero-fill the declared size (up to 1 TiB)
    before decompressing."""
    return pos if codec == 0 or pos < 3 or pos >= 8 else 8


def mutate(rng, wire):
    """One seeded mutation of a PULP file; returns (kind, bytes)."""
    hdr, blobs = parse_layout(wire)
    codec = hdr["codec"]
    T = len(blobs)
    body0 = len(wire) - sum(len(i) + len(v) for i, v in blobs)
    k = int(rng.integers(0, 14))
    w = bytearray(wire)
    if T == 0 or k == 0:  # truncation anywhere
        return "truncate", bytes(w[: int(rng.integers(0, len(w)))])
    t = int(rng.integers(0, T))
    ib, vb = blobs[t]
    if k in (1, 2) and ib:  # bit flips in an index blob
        b = bytearray(ib)
        for _ in range(int(rng.integers(1, 4))):
            p = _guard(int(rng.integers(0, len(b))), codec)
            if p < len(b):
                b[p] ^= 1 << int(rng.integers(0, 8))
        blobs[t][0] = bytes(b)
        return "index_flip", assemble(hdr, blobs)
    if k == 3 and ib:  # 0xFF / 0xFFFF marker runs
        b = bytearray(ib)
        p = _guard(int(rng.integers(0, len(b))), codec)
        run = int(rng.choice([1, 2, 3, 4, 5, 6, 8])) if codec == 0 else 1
        b[p:p + run] = b"\xff" * len(b[p:p + run])
        blobs[t][0] = bytes(b)
        return "marker_run", assemble(hdr, blobs)
    if k == 4 and ib:  # zeroed gap bytes
        b = bytearray(ib)
        p = _guard(int(rng.integers(0, len(b))), codec)
        n = int(rng.integers(1, 5)) if codec == 0 else 1
        b[p:p + n] = b"\0" * len(b[p:p + n])
        blobs[t][0] = bytes(b)
        return "zero_run", assemble(hdr, blobs)
    if k == 5:  # count edit, value blob resized to match
        d = int(rng.choice([-3, -1, 1, 2, 7]))
        c = max(0, hdr["tensors"][t]["count"] + d)
        hdr["tensors"][t]["count"] = c
        hdr["tensors"][t]["value_nbytes"] = 2 * c
        blobs[t][1] = (vb + bytes(rng.integers(0, 256, 16, dtype=np.uint8)))[: 2 * c] if hdr["codec"] == 0 else vb
        return "count_edit", assemble(hdr, blobs)
    if k == 6:  # index_nbytes edit, index blob resized (extra bytes or cut)
        d = int(rng.choice([-4, -2, -1, 1, 2, 3, 5]))
        n = max(0, len(ib) + d)
        blobs[t][0] = (ib + bytes(rng.integers(0, 256, 8, dtype=np.uint8)))[:n]
        hdr["tensors"][t]["index_nbytes"] = n
        return "index_nbytes_edit", assemble(hdr, blobs)
    if k == 7:  # value_nbytes disagrees with count (blob resized, count kept)
        d = int(rng.choice([-2, -1, 1, 2]))
        n = max(0, len(vb) + d)
        blobs[t][1] = (vb + b"\x11\x22")[:n]
        hdr["tensors"][t]["value_nbytes"] = n
        return "value_nbytes_edit", assemble(hdr, blobs)
    if k == 8:  # duplicate tensor: same entry and blobs again, right after (last one wins in decode)
        e = dict(hdr["tensors"][t])
        if rng.random() < 0.5 and vb:  # the duplicate carries different values
            vb2 = bytearray(vb)
            p = _guard(int(rng.integers(0, len(vb2))), codec)
            if p < len(vb2):
                vb2[p] ^= 0x40
            vb = bytes(vb2)
        hdr["tensors"].insert(t + 1, e)
        blobs.insert(t + 1, [ib, vb])
        return "duplicate", assemble(hdr, blobs)
    if k == 9 and T > 1:  # unsorted names: swap two entries with their blobs
        u = int(rng.integers(0, T))
        hdr["tensors"][t], hdr["tensors"][u] = hdr["tensors"][u], hdr["tensors"][t]
        blobs[t], blobs[u] = blobs[u], blobs[t]
        return "swap", assemble(hdr, blobs)
    if k == 10:  # shape edit (last extent or rank)
        shp = list(hdr["tensors"][t]["shape"])
        c = int(rng.integers(0, 4))
        if c == 0:
            shp[-1] = max(1, shp[-1] + int(rng.choice([-1, 1, 5])))
        elif c == 1:
            shp = [int(np.prod(shp))]
        elif c == 2:
            shp = shp + [1]
        else:
            shp[0] = int(rng.choice([0, -1, 1]))
        hdr["tensors"][t]["shape"] = shp
        return "shape_edit", assemble(hdr, blobs)
    if k == 11 and vb:  # value bit flips (read succeeds; decode's hash check fails)
        b = bytearray(vb)
        p = _guard(int(rng.integers(0, len(b))), codec)
        if p < len(b):
            b[p] ^= 1 << int(rng.integers(0, 8))
        blobs[t][1] = bytes(b)
        return "value_flip", assemble(hdr, blobs)
    if k == 12:  # unknown tensor name / header field edits
        c = int(rng.integers(0, 5))
        if c == 0:
            hdr["tensors"][t]["name"] = hdr["tensors"][t]["name"] + "_x"
        elif c == 1:
            hdr["target_step"] = hdr["target_step"] + 1
        elif c == 2:
            hdr["codec"] = int(rng.choice([5, 9]))
        elif c == 3:
            hdr["representation"] = "COO_INT64"
        else:
            hdr["tensors"][t].pop(str(rng.choice(["count", "index_nbytes", "value_nbytes", "shape", "name"])))
        return "header_field", assemble(hdr, blobs)
    # header byte noise (JSON syntax / schema errors) and whole-file bit flips
    p = int(rng.integers(0, body0 if (rng.random() < 0.7 or codec != 0) else len(w)))
    w[p] = int(rng.integers(0, 256))
    return "byte_noise", bytes(w)


def outcome(fn):
    from paper_2602_03839_b200._native import PulseError
    try:
        return ("ok", fn())
    except OracleError as e:
        return (e.kind, e.msg)
    except PulseError as e:
        return (e.kind, str(e).split(": ", 1)[1] if ": " in str(e) else "")


def same_patch(a, b):
    if (a.base_step, a.target_step, a.anchor_step, a.representation, a.codec, bytes(a.target_hash)) != \
            (b.base_step, b.target_step, b.anchor_step, b.representation, b.codec, bytes(b.target_hash)):
        return False
    if len(a.tensors) != len(b.tensors):
        return False
    for x, y in zip(a.tensors, b.tensors):
        if x.name != y.name or tuple(x.shape) != tuple(y.shape):
            return False
        if not (np.array_equal(x.indices, y.indices) and np.array_equal(x.values, y.values)):
            return False
    return True


def test_fuzzed_pulp_files_match_reference(golden):
    from oracle.oracle import Patch, TensorPatch
    R = reference()
    H = _H()
    rng = np.random.default_rng(20261019)
    corpus = []
    for name in CASES:
        prev, curr, _ = golden.case(name)
        for r in (0, 1, 2):
            for codec in (0, 0, 0, 2, 1, 4):  # identity weighted: the device decoders see raw payloads
                wire = golden.pulp(name, r, codec)
                if wire is not None:
                    corpus.append((name, r, codec, prev, wire))
    mismatches, kinds = [], {}
    resident_checked = 0
    for i in range(N_MUTATIONS):
        name, r, codec, prev, wire = corpus[int(rng.integers(0, len(corpus)))]
        kind, m = mutate(rng, wire)
        kinds[kind] = kinds.get(kind, 0) + 1
        ref = outcome(lambda: R.read_patch_bytes(m))
        ours = outcome(lambda: H.read_patch_bytes(m))
        rec = {"i": i, "case": name, "repr": r, "codec": codec, "kind": kind}
        if ref[0] != ours[0] or (ref[0] != "ok" and ref[1] != ours[1]):
            mismatches.append({**rec, "stage": "read", "ref": list(ref), "ours": list(ours), "hex": m.hex()})
            continue
        if ref[0] == "ok" and not same_patch(ref[1], ours[1]):
            mismatches.append({**rec, "stage": "read-content", "hex": m.hex()})
            continue
        if ref[0] == "ok":
            rd = outcome(lambda: R.decode(prev, ref[1], verify=True))
            od = outcome(lambda: H.decode(_mirror(prev), ours[1], verify_hash=True))
            if rd[0] != od[0] or (rd[0] != "ok" and rd[1] != od[1]):
                mismatches.append({**rec, "stage": "decode", "ref": list(rd), "ours": list(od), "hex": m.hex()})
                continue
            if rd[0] == "ok":
                got = {t.name: t.data for t in od[1].tensors}
                if any(not np.array_equal(t.data, got[t.name]) for t in rd[1].tensors):
                    mismatches.append({**rec, "stage": "decode-content", "hex": m.hex()})
                    continue
        else:
            rd = None
        if i % 25 == 0:  # apply_delta on a resident copy of the base
            resident_checked += 1
            res = H.Resident(_mirror(prev))
            ra = outcome(lambda: res.apply(m, 1, verify=True))
            if ref[0] != "ok":
                want = ref[0]
            elif ref[1].base_step != 0 or ref[1].target_step != 1:
                want = "ProtocolViolationError"
            else:
                want = rd[0]
            after = res.download()
            if ra[0] != want:
                mismatches.append({**rec, "stage": "resident", "ref": want, "ours": list(ra), "hex": m.hex()})
            elif want == "ok":
                got = {t.name: t.data for t in after.tensors}
                if any(not np.array_equal(t.data, got[t.name]) for t in rd[1].tensors) or res.step != 1:
                    mismatches.append({**rec, "stage": "resident-content", "hex": m.hex()})
            elif res.step != 0 or any(not np.array_equal(a.data, b.data) for a, b in zip(after.tensors, prev.tensors)):
                mismatches.append({**rec, "stage": "resident-untouched", "hex": m.hex()})
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "fuzz_mismatches.json"), "w") as f:
        json.dump({"n": N_MUTATIONS, "kinds": kinds, "resident_checked": resident_checked,
                   "mismatches": mismatches[:400], "n_mismatches": len(mismatches)}, f, indent=1)
    summary = {}
    for x in mismatches:
        summary[(x["kind"], x["stage"])] = summary.get((x["kind"], x["stage"]), 0) + 1
    assert not mismatches, f"{len(mismatches)} of {N_MUTATIONS} mutations disagree with the reference: {summary}"
