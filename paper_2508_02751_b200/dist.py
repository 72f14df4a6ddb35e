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
  * heads + partitioned SLM (NEXT f3b): as heads, but the SLM rows are split
    too — rank r scores and selects only the flat SLM heads [j0, j1) of its
    block (`slm_row_block`), the ranks all-gather the compact selection lists
    of their blocks (`exchange_selection`), then every rank plans and attends
    its kv-groups with the full selection.  This lifts the replicated-SLM cap of
    head sharding at the price of one more all-gather per step.
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


# --------------------------------------------------------------------------- f3b
def slm_row_block(n_slm: int, world: int, rank: int) -> Tuple[int, int]:
    """Flat SLM heads [j0, j1) scored and selected by `rank` (contiguous,
    equal-sized blocks except the last)."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    per = -(-n_slm // world)
    return min(rank * per, n_slm), min((rank + 1) * per, n_slm)


def select_head_map(head_map: torch.Tensor, j0: int, j1: int) -> torch.Tensor:
    """The entries of a head map whose SLM row lies in [j0, j1): passed to
    smallkv_select as its head map, it makes the kernel score and split exactly
    the image rows of the block (the ABI derives the row set from the map)."""
    hm = head_map.reshape(-1)
    return hm[(hm >= j0) & (hm < j1)].contiguous()


SELECTION_FIELDS = ("lse", "crit", "marg", "marg_w", "counts")


def exchange_selection(out, n_slm: int, group=None):
    """All-gather the per-rank blocks of the selection outputs (indexed by flat
    SLM head along dim 0: lse, crit, marg, marg_w, counts) so that every rank
    holds every row; rank r contributes rows slm_row_block(n_slm, w, r) of its
    own tensors (other rows are overwritten)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_slm // world)
    for name in SELECTION_FIELDS:
        t = getattr(out, name)
        tail = t.shape[1:]
        local = torch.zeros((per,) + tuple(tail), dtype=t.dtype, device=t.device)
        j0, j1 = slm_row_block(n_slm, world, rank)
        local[: j1 - j0] = t[j0:j1]
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local, group=group)
        full = torch.cat(parts, dim=0)[:n_slm]
        t.copy_(full)
    return out


def exchange_bytes(out, n_slm: int, world: int) -> int:
    """Bytes each rank receives per step in exchange_selection."""
    per = -(-n_slm // world)
    tot = 0
    for name in SELECTION_FIELDS:
        t = getattr(out, name)
        tot += per * (world - 1) * t[0].numel() * t.element_size()
    return tot
