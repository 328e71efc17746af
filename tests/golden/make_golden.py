"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs the unmodified reference (oracle/_ref/libpulse_ref.so, built by
`make -C oracle` from /root/reference/proj/include) on small seeded inputs and
records inputs plus the reference's outputs:

  synth_cases.npz   prev/curr snapshots of each case (uint16 bit patterns)
  patches.npz       PULP bytes for every (case, representation, codec)
  golden.json       manifest: specs, change counts, target hashes, sizes,
                    and the config-1 (16M, seed 7) summary numbers

Usage:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Checkpoint, Tensor, reference, IDENTITY, LZ4, ZSTD1, ZSTD3, GZIP6  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, shapes, sparsity, cluster_width, seed)
CASES = [
    # test_patch.cpp:92-108 roundtrip spec
    *[(f"roundtrip_s{s}", [(64, 96), (1000,), (7, 11, 13)], 0.97, 16, s) for s in range(5)],
    # test_patch_file.cpp:45-56 sample_patch spec
    *[(f"patchfile_s{s}", [(48, 32), (700,)], 0.96, 8, s) for s in (1, 2, 3)],
    # acceptance.cpp:54-60 shape families at several sparsities / widths
    ("accept_a", [(48, 32), (640,)], 0.5, 1, 1000),
    ("accept_b", [(2048,), (16, 8, 8)], 0.9, 8, 1001),
    ("accept_c", [(48, 32), (640,)], 0.999, 256, 1002),
    ("dense_all", [(33, 7)], 0.0, 1, 2),
    # escape-heavy: very sparse wide rows -> row gaps >= 255 and col entries >= 65535
    ("esc_rows", [(20000, 3)], 0.9995, 1, 5),
    ("esc_cols", [(300000,)], 0.99995, 1, 6),
    ("esc_cols_wide", [(2, 140000)], 0.99998, 1, 9),
]


def handcrafted(Checkpoint, Tensor):
    """Zero base with changes placed to hit every escape path, including
    escape payloads that contain the 0xFF / 0xFFFF marker bytes
    (index_coding.hpp:59-100)."""
    a = np.zeros(140000 * 2, np.uint16)     # row gaps 255, 511, 65535, 65536
    for r in [0, 255, 766, 66301, 131837]:
        a[r * 2] = 0x3F80
        a[r * 2 + 1] = 0x0001
    b = np.zeros(300000, np.uint16)         # one row: col entries 65535, 0x1FFFF, 0xFFFF+...
    for c in [3, 3 + 65535, 3 + 65535 + 0x1FFFF, 299999]:
        b[c] = 0x8000
    c = np.zeros(7 * 11 * 13, np.uint16)
    c[::3] = 0x7FC0
    prev = Checkpoint(0, [Tensor("a.rows", (140000, 2), np.zeros_like(a)),
                          Tensor("b.cols", (300000,), np.zeros_like(b)),
                          Tensor("c.dense", (7, 11, 13), np.zeros_like(c))])
    curr = Checkpoint(1, [Tensor("a.rows", (140000, 2), a), Tensor("b.cols", (300000,), b),
                          Tensor("c.dense", (7, 11, 13), c)])
    return prev, curr


def h5_unchanged(Checkpoint, Tensor):
    """FLAT_INT32 gap bases when unchanged tensors sit before and between
    changed ones (patch.hpp:131-156: the base advances only over tensors the
    patch carries, and encode omits unchanged tensors, patch.hpp:302-304).
    Name order: a.lead (unchanged), b.changed, c.mid (unchanged), d.changed,
    e.tail (unchanged)."""
    rng = np.random.default_rng(55)
    shapes = {"a.lead": (300, 7), "b.changed": (64, 33), "c.mid": (5000,), "d.changed": (17, 19, 3),
              "e.tail": (129,)}
    prev, curr = [], []
    for name, shp in shapes.items():
        n = int(np.prod(shp))
        a = rng.integers(0, 65536, n, dtype=np.uint16)
        b = a.copy()
        if "changed" in name:
            b[rng.random(n) < 0.05] ^= 1
            b[0 if name.startswith("d") else n - 1] ^= 0x8000   # first element of d, last of b
        prev.append(Tensor(name, shp, a))
        curr.append(Tensor(name, shp, b))
    return Checkpoint(0, prev), Checkpoint(1, curr)


def h5_sparse_lead(Checkpoint, Tensor):
    """A large unchanged leading tensor, then changed tensors separated by
    unchanged ones (counting their numel into the base would shift every later gap)."""
    rng = np.random.default_rng(56)
    shapes = [("m.a", (70000,)), ("m.b", (40, 40)), ("m.c", (200000,)), ("m.d", (3, 5)), ("m.e", (8, 8)),
              ("m.f", (2000,))]
    changed = {"m.b", "m.d", "m.f"}
    prev, curr = [], []
    for name, shp in shapes:
        n = int(np.prod(shp))
        a = rng.integers(0, 65536, n, dtype=np.uint16)
        b = a.copy()
        if name in changed:
            b[rng.choice(n, max(1, n // 20), replace=False)] ^= 1
        prev.append(Tensor(name, shp, a))
        curr.append(Tensor(name, shp, b))
    return Checkpoint(0, prev), Checkpoint(1, curr)


HANDCRAFTED = {"handcrafted": handcrafted, "h5_unchanged": h5_unchanged, "h5_sparse_lead": h5_sparse_lead}

# Spec-only cases at real Qwen2.5-7B tensor shapes: the inputs are too large to
# store, so the tests regenerate them with the reference generator
# (oracle/_ref, draw for draw) and check the stored target hash first.  Only
# the identity-codec PULP bytes are kept (large.npz).
LARGE = [
    # 99.99% on mlp.gate_proj [18944, 3584]: sparse enough that row gaps reach
    # 255 and COO_DOWNSCALED emits 0xFF + u32 row escapes
    ("s7b_9999", [(18944, 3584), (3584,), (512,)], 0.9999, 64, 77),
    # 99% on the same tensors: the headline sparsity, no escapes
    ("s7b_99", [(18944, 3584), (3584,), (512,)], 0.99, 64, 78),
]

CODECS = [IDENTITY, LZ4, ZSTD1, ZSTD3, GZIP6]


def main():
    R = reference()
    snaps, patches, manifest = {}, {}, {"cases": {}}
    for name, shapes, sp, cw, seed in CASES + [(h, None, None, None, None) for h in HANDCRAFTED]:
        if shapes is None:
            prev, curr = HANDCRAFTED[name](Checkpoint, Tensor)
            shapes = [t.shape for t in prev.tensors]
        else:
            prev, curr = R.generate_synthetic(shapes, sp, cw, seed)
        for i, (a, b) in enumerate(zip(prev.tensors, curr.tensors)):
            snaps[f"{name}/prev/{i}"] = a.data
            snaps[f"{name}/curr/{i}"] = b.data
        entry = {"shapes": [list(s) for s in shapes], "sparsity": sp, "cluster_width": cw,
                 "seed": seed, "names": [t.name for t in prev.tensors],
                 "target_hash": R.hash_weights(curr).hex(), "patches": {}}
        for r in (0, 1, 2):
            for c in CODECS:
                try:
                    p = R.encode(curr, prev, r, c)
                    wire = R.write_patch_bytes(p)
                except Exception as e:  # recorded so tests can expect the same error
                    entry["patches"][f"{r}/{c}"] = {"error": str(e)}
                    continue
                patches[f"{name}/{r}/{c}"] = np.frombuffer(wire, np.uint8)
                entry["patches"][f"{r}/{c}"] = {"nbytes": len(wire), "changes": p.total_changes()}
        manifest["cases"][name] = entry
        print(name, entry["patches"]["0/0"])

    # Config 1 (BASELINE.json configs[0]): 4096^2, 99%, cluster 64, seed 7.
    prev, curr = R.generate_synthetic([(4096, 4096)], 0.99, 64, 7)
    c1 = {"changes": None, "target_hash": R.hash_weights(curr).hex(), "pulp_nbytes": {}}
    for r in (0, 1, 2):
        for c in CODECS:
            p = R.encode(curr, prev, r, c)
            c1["changes"] = p.total_changes()
            c1["pulp_nbytes"][f"{r}/{c}"] = len(R.write_patch_bytes(p))
    manifest["config1"] = c1
    print("config1", c1)

    large, large_bytes = {}, {}
    for name, shapes, sp, cw, seed in LARGE:
        prev, curr = R.generate_synthetic(shapes, sp, cw, seed)
        p = R.encode(curr, prev, 0, IDENTITY)
        entry = {"shapes": [list(s) for s in shapes], "sparsity": sp, "cluster_width": cw, "seed": seed,
                 "names": [t.name for t in prev.tensors], "prev_hash": R.hash_weights(prev).hex(),
                 "target_hash": R.hash_weights(curr).hex(), "changes": p.total_changes(), "pulp_nbytes": {}}
        for r in (0, 1, 2):
            p.representation = r
            wire = R.write_patch_bytes(p)
            if len(wire) <= (256 << 10):  # small enough to keep; larger ones by digest
                large_bytes[f"{name}/{r}"] = np.frombuffer(wire, np.uint8)
            entry["pulp_nbytes"][str(r)] = len(wire)
            entry.setdefault("pulp_sha256", {})[str(r)] = R.sha256(wire).hex()
        large[name] = entry
        print(name, entry["changes"], entry["pulp_nbytes"])
    manifest["large"] = large
    np.savez_compressed(os.path.join(HERE, "large.npz"), **large_bytes)

    np.savez_compressed(os.path.join(HERE, "synth_cases.npz"), **snaps)
    np.savez_compressed(os.path.join(HERE, "patches.npz"), **patches)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
