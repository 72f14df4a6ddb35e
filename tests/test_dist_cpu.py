"""World-size-2 gloo tests of the multi-GPU host logic (CPU only)."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_02751_b200 import dist as pdist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # max over ranks of a per-rank timing
        m = pdist.max_over_ranks(10.0 + rank)
        # head-split gather: rank r holds heads [r*Hl, (r+1)*Hl) of a known tensor
        B, H, d = 3, 8, 5
        full = torch.arange(B * H * d, dtype=torch.float32).view(B, H, d)
        Hl = H // world
        local = full[:, rank * Hl:(rank + 1) * Hl]
        gathered = pdist.gather_heads(local)
        q.put((rank, m, torch.equal(gathered, full)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, ok in res:
        assert m == 11.0 and ok


@pytest.mark.parametrize("B,w", [(32, 2), (8, 8), (7, 2), (5, 4)])
def test_batch_shards_partition(B, w):
    got = sorted(b for r in range(w) for b in pdist.batch_shard(B, w, r))
    assert got == list(range(B))
    sizes = [len(pdist.batch_shard(B, w, r)) for r in range(w)]
    assert max(sizes) - min(sizes) <= 1


def test_kv_group_ranges_and_head_map_slice():
    L, H, Hkv = 3, 8, 4
    hm = torch.arange(L * H, dtype=torch.int32)
    parts = []
    for r in range(2):
        g0, g1 = pdist.kv_group_range(Hkv, 2, r)
        assert (g0, g1) == (2 * r, 2 * r + 2)
        parts.append(pdist.head_map_slice(hm, L, H, Hkv, g0, g1).view(L, -1))
    assert torch.equal(torch.cat(parts, dim=1).view(-1), hm)
    with pytest.raises(ValueError):
        pdist.kv_group_range(6, 4, 0)
