"""Test-side helpers: de-paging and brute-force references (no method code).

These re-derive inputs for library routines (torch SDPA / softmax / matmul,
Python `sorted`) that pin the oracle; they never call the CUDA path.
"""
from __future__ import annotations

import numpy as np
import torch


def dense_rows(cache, layer_slot: int, b: int, n: int, kvh: int, which: str = "k") -> torch.Tensor:
    """Logical [n, d] rows of (layer slot, sequence b, kv head) as fp64 CPU."""
    pool = cache.k if which == "k" else cache.v
    ps = cache.page_size
    pos = torch.arange(n)
    pages = cache.block_table[b].cpu().long()[pos // ps]
    rows = pool[layer_slot].cpu()[pages, kvh, pos % ps]  # [n, d]
    return rows.double()


def brute_split(score, K: int, R: int, M: int):
    """Definition of the split by a full Python sort (P5): recent = last R',
    rank the rest by (score desc, index asc), crit = first K', marg = next M'."""
    n = len(score)
    Rc = min(R, n)
    Kc = min(K, n - Rc)
    Mc = min(M, n - Rc - Kc)
    order = sorted(range(n - Rc), key=lambda v: (-score[v], v))
    crit = sorted(order[:Kc])
    marg = sorted(order[Kc:Kc + Mc])
    recent = list(range(n - Rc, n))
    evicted = sorted(order[Kc + Mc:])
    return crit, marg, recent, evicted


def sdpa_fp64(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, mask=None) -> torch.Tensor:
    """torch scaled_dot_product_attention in fp64 for one query vector."""
    qq = q.double().view(1, 1, 1, -1)
    kk = K.double().view(1, 1, K.shape[0], -1)
    vv = V.double().view(1, 1, V.shape[0], -1)
    m = None if mask is None else torch.as_tensor(mask, dtype=torch.bool).view(1, 1, 1, -1)
    return torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, attn_mask=m).view(-1)


def row_normwise_err(o: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """max_i |o - ref| / max_i |ref| per leading index (A19 metric)."""
    num = np.abs(o - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-30)
    return num / den
