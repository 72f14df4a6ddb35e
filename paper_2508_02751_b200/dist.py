"""Multi-GPU partitioning of the decode hot path (host logic + torch.distributed).

Two partitions shard the path without changing any kernel (SURVEY §8(e),
DESIGN.md §9):
  * batch: rank r owns sequences {b : b mod world == r} with both models'
    caches for them; no collective on the data path (weak scaling).
  * heads: rank r owns LLM kv-groups [r*H_kv/w, (r+1)*H_kv/w) of every layer
    for all sequences; it runs smallkv_select for the SLM rows its heads map
    to (the SLM cache is replicated) and smallkv_attend on its kv-head slice,
    then the per-head outputs [B, H/w, d] are all-gathered (NCCL over NVLink)
    into [B, H, d] — the only exchange step of the path.
Every rank's results are bit-identical to the unsharded run (the kernels are
deterministic and per-(sequence, kv-group) work does not depend on neighbours).
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def batch_shard(global_batch: int, world: int, rank: int) -> List[int]:
    """Sequences owned by `rank` (round-robin, so ragged batches stay balanced)."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    return list(range(rank, global_batch, world))


def kv_group_range(num_kv_heads: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous kv-group range [g0, g1) owned by `rank` in head-split mode."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} kv-heads do not split over {world} ranks")
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per


def head_map_slice(head_map: torch.Tensor, layers: int, q_heads: int, kv_heads: int,
                   g0: int, g1: int) -> torch.Tensor:
    """Rows of the [L*H] head map for the q-heads of kv-groups [g0, g1), as the
    [L*(H_loc)] map of a model whose layer has only those heads."""
    G = q_heads // kv_heads
    hm = head_map.view(layers, q_heads)[:, g0 * G:g1 * G]
    return hm.contiguous().view(-1)


def gather_heads(local_out: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-rank head slices [..., H_loc, d] into [..., H, d] (rank
    order = head order)."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local_out) for _ in range(world)]
    dist.all_gather(parts, local_out.contiguous(), group=group)
    return torch.cat(parts, dim=-2)


def max_over_ranks(value: float, device: Optional[torch.device] = None, group=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the slowest rank)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def slice_llm_kv_groups(k: torch.Tensor, v: torch.Tensor, q: torch.Tensor,
                        head_map: torch.Tensor, layers: int, q_heads: int, kv_heads: int,
                        g0: int, g1: int):
    """Head-split shard of the LLM side: pools [Lc][pages][H_kv][ps][d] -> kv-heads
    [g0, g1); queries [..][B][H][d] -> the groups' q-heads; the head map sliced
    accordingly.  (A real deployment allocates only its slice; this copies.)"""
    G = q_heads // kv_heads
    return (k[:, :, g0:g1].contiguous(), v[:, :, g0:g1].contiguous(),
            q[..., g0 * G:g1 * G, :].contiguous(),
            head_map_slice(head_map, layers, q_heads, kv_heads, g0, g1))
