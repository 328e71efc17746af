"""CPU coverage of the multi-GPU host logic: shard bounds, FLAT carry, section
offsets, and the collectives (size exchange, section gather) over a
world_size-2 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_03839_b200.shapes import QWEN, numel, qwen_state_dict, shard
from paper_2602_03839_b200 import shard as S

SUMMARY_DTYPE = np.dtype([("n_changes", "<u8"), ("has_change", "<u8"), ("last_gap_base", "<u8"), ("status", "<u8")])


@pytest.mark.parametrize("model", sorted(QWEN))
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_shard_bounds_cover_name_order(model, n):
    sd = qwen_state_dict(model)
    assert [x[0] for x in sd] == sorted(x[0] for x in sd)  # bytewise name order (checkpoint.hpp:74-80)
    b = shard(sd, n)
    assert len(b) == n + 1 and b[0] == 0 and b[-1] == len(sd)
    assert all(b[i] <= b[i + 1] for i in range(n))
    loads = [sum(numel(s) for _, s in sd[b[i]:b[i + 1]]) for i in range(n)]
    biggest = max(numel(s) for _, s in sd)
    assert max(loads) <= max(biggest, sum(loads) / n + biggest)


def test_qwen_element_counts():
    # counts quoted in SURVEY 8(d)
    assert sum(numel(s) for _, s in qwen_state_dict("qwen2.5-7b")) == 7_615_616_512
    assert sum(numel(s) for _, s in qwen_state_dict("qwen2.5-1.5b")) == 1_543_714_304
    assert sum(numel(s) for _, s in qwen_state_dict("qwen2.5-32b")) == 32_763_876_352
    assert len(qwen_state_dict("qwen2.5-7b")) == 339


def test_flat_carry_picks_nearest_earlier_rank_with_changes():
    s = np.zeros(4, SUMMARY_DTYPE)
    s["has_change"] = [1, 0, 1, 1]
    s["last_gap_base"] = [10, 0, 30, 40]
    assert S.flat_carry(s, 0) == (0, 0)
    assert S.flat_carry(s, 1) == (1, 10)
    assert S.flat_carry(s, 2) == (1, 10)   # rank 1 emitted nothing
    assert S.flat_carry(s, 3) == (1, 30)


def test_section_offsets():
    bo, eo = S.section_offsets([5, 0, 7], [2, 0, 3])
    assert bo.tolist() == [0, 5, 5] and eo.tolist() == [0, 2, 2]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes = [3, 5]
        bb, ne = S.exchange_sizes(sizes[rank], rank + 1, torch.device("cpu"))
        section = torch.arange(sizes[rank], dtype=torch.uint8) + 10 * rank
        full = S.gather_sections(section, bb, root=0)
        q.put((rank, bb.tolist(), ne.tolist(), None if full is None else full.tolist()))
    finally:
        dist.destroy_process_group()


def test_exchange_and_gather_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict((r, (bb, ne, full)) for r, bb, ne, full in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
    assert out[0][0] == [3, 5] and out[1][0] == [3, 5]
    assert out[0][1] == [1, 2]
    assert out[0][2] == [0, 1, 2, 10, 11, 12, 13, 14]
    assert out[1][2] is None
