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


def _exchange_worker(rank: int, world: int, port: int, q):
    import types
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_slm, B = 7, 3
        g = torch.Generator().manual_seed(5)
        ref = types.SimpleNamespace(
            lse=torch.randn(n_slm, B, 2, generator=g),
            crit=torch.randint(0, 99, (n_slm, B, 4), generator=g, dtype=torch.int32),
            marg=torch.randint(0, 99, (n_slm, B, 5), generator=g, dtype=torch.int32),
            marg_w=torch.rand(n_slm, B, 5, generator=g),
            counts=torch.randint(0, 4, (n_slm, B, 2), generator=g, dtype=torch.int32))
        # each rank only computed its own block; other rows hold garbage
        mine = types.SimpleNamespace(**{k: torch.full_like(v, -7) for k, v in vars(ref).items()})
        j0, j1 = pdist.slm_row_block(n_slm, world, rank)
        for k in vars(ref):
            getattr(mine, k)[j0:j1] = getattr(ref, k)[j0:j1]
        pdist.exchange_selection(mine, n_slm)
        ok = all(torch.equal(getattr(mine, k), getattr(ref, k)) for k in vars(ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_f3b_slm_row_blocks_and_selection_exchange():
    """f3b host logic: SLM row blocks partition [0, n_slm); the head-map subset
    of a block maps only into it; after the gloo all-gather every rank holds
    every row of the selection outputs."""
    for n_slm, w in [(7, 2), (336, 4), (3, 8)]:
        blocks = [pdist.slm_row_block(n_slm, w, r) for r in range(w)]
        cover = [j for a, b in blocks for j in range(a, b)]
        assert cover == list(range(n_slm))
    hm = torch.tensor([5, 0, 6, 2, 2, 3], dtype=torch.int32)
    assert pdist.select_head_map(hm, 0, 3).tolist() == [0, 2, 2]
    assert pdist.select_head_map(hm, 3, 7).tolist() == [5, 6, 3]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok in res), res
