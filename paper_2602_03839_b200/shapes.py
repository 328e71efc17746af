"""State-dict shapes for the benchmark workloads (BASELINE.json configs).

Qwen2.5 shapes follow the public model configs (hidden / intermediate /
layers / heads / kv heads / vocab; q,k,v biases; 1.5B ties embeddings, 7B and
32B do not).  They are not part of the reference; they fix the tensor table
the benchmark runs on.  Tensors are returned in ascending bytewise name order
-- the order PULSE hashes and serializes them (checkpoint.hpp:74-80,
patch_file.hpp:34-35).
"""
from __future__ import annotations

QWEN = {
    # name: (hidden, intermediate, layers, heads, kv_heads, vocab, tied)
    "qwen2.5-1.5b": (1536, 8960, 28, 12, 2, 151936, True),
    "qwen2.5-7b": (3584, 18944, 28, 28, 4, 152064, False),
    "qwen2.5-32b": (5120, 27648, 64, 40, 8, 152064, False),
}


def qwen_state_dict(model: str):
    """[(name, shape)] of a Qwen2.5 bf16 state dict, name-sorted."""
    h, inter, layers, heads, kv, vocab, tied = QWEN[model]
    hd = h // heads
    kvd = kv * hd
    out = [("model.embed_tokens.weight", (vocab, h)), ("model.norm.weight", (h,))]
    if not tied:
        out.append(("lm_head.weight", (vocab, h)))
    for i in range(layers):
        p = f"model.layers.{i}."
        out += [
            (p + "input_layernorm.weight", (h,)),
            (p + "post_attention_layernorm.weight", (h,)),
            (p + "self_attn.q_proj.weight", (h, h)), (p + "self_attn.q_proj.bias", (h,)),
            (p + "self_attn.k_proj.weight", (kvd, h)), (p + "self_attn.k_proj.bias", (kvd,)),
            (p + "self_attn.v_proj.weight", (kvd, h)), (p + "self_attn.v_proj.bias", (kvd,)),
            (p + "self_attn.o_proj.weight", (h, h)),
            (p + "mlp.gate_proj.weight", (inter, h)),
            (p + "mlp.up_proj.weight", (inter, h)),
            (p + "mlp.down_proj.weight", (h, inter)),
        ]
    return sorted(out, key=lambda x: x[0].encode())


def numel(shape) -> int:
    n = 1
    for x in shape:
        n *= int(x)
    return n


def workload(name: str):
    """Named workloads: 'c1' (BASELINE configs[0]: one 4096x4096 tensor),
    'c1-flat' (the same as rank-1), or a Qwen2.5 model."""
    if name == "c1":
        return [("tensor_00", (4096, 4096))]
    if name == "c1-flat":
        return [("tensor_00", (4096 * 4096,))]
    return qwen_state_dict(name)


def shard(tensors, n_ranks: int):
    """Contiguous ranges of the name-sorted tensor list that
    minimise the largest shard (linear partition: binary search on the load
    bound, greedy packing).  Rank r gets tensors [bounds[r], bounds[r+1]);
    the rank-major concatenation of per-rank patch sections is the full PULP
    body, because PULP orders tensors by name (patch_file.hpp:34-35)."""
    sizes = [numel(s) for _, s in tensors]

    def pack(limit):
        bounds, acc = [0], 0
        for i, n in enumerate(sizes):
            if acc + n > limit and acc > 0:
                bounds.append(i)
                acc = 0
            acc += n
        return bounds

    lo, hi = max(sizes) if sizes else 0, sum(sizes)
    while lo < hi:
        mid = (lo + hi) // 2
        if len(pack(mid)) <= n_ranks:
            hi = mid
        else:
            lo = mid + 1
    bounds = pack(lo)
    while len(bounds) < n_ranks:  # fewer non-empty shards than ranks: trailing ranks get nothing
        bounds.append(len(tensors))
    return bounds + [len(tensors)]
