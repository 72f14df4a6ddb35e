"""Algorithmic byte model of the decode hot path (host logic, no kernels).

Eq. 7 (App. A): M_kv = 2 L N_kv D_kv S B C_b.  The per-step bytes
the path must touch are the full SLM K cache (R11) plus,
per LLM layer, the critical ∪ recent K+V rows and the marginal-only V rows,
counted once per (sequence, kv-group).
"""
from __future__ import annotations

from typing import Sequence, Tuple

BF16 = 2


def kv_cache_bytes(L: int, N_kv: int, D_kv: int, S: int, B: int, C_b: int = BF16) -> int:
    """Eq. 7: bytes of a full K+V cache."""
    return 2 * L * N_kv * D_kv * S * B * C_b


def clamp_budget(n: int, K: int, R: int, M: int) -> Tuple[int, int, int]:
    """R' = min(R,n), K' = min(K,n-R'), M' = min(M,n-R'-K') (R5)."""
    Rc = max(0, min(R, n))
    Kc = max(0, min(K, n - Rc))
    Mc = max(0, min(M, n - Rc - Kc))
    return Kc, Rc, Mc


def slm_score_bytes(slm_layers: int, slm_kv_heads: int, slm_head_dim: int,
                    seq_lens: Sequence[int]) -> int:
    """K1: every SLM layer's K' over every sequence's full context."""
    return sum(slm_layers * slm_kv_heads * n * slm_head_dim * BF16 for n in seq_lens)


def attend_bytes_coherent(kv_heads: int, head_dim: int, seq_lens: Sequence[int],
                          budgets: Sequence[Tuple[int, int, int]]) -> int:
    """K3 for one LLM layer when every q-head of a kv-group shares one SLM row
    (the group's union is one set): (K'+R') K+V rows + M' V rows per group."""
    tot = 0
    for n, (K, R, M) in zip(seq_lens, budgets):
        Kc, Rc, Mc = clamp_budget(n, K, R, M)
        tot += kv_heads * ((Kc + Rc) * 2 * head_dim * BF16 + Mc * head_dim * BF16)
    return tot


def step_bytes_coherent(cfg, seq_lens: Sequence[int], budgets, llm_layers: int) -> dict:
    """Per-step algorithmic bytes: select (all SLM layers) + llm_layers attends."""
    s = slm_score_bytes(cfg.slm.layers, cfg.slm.kv_heads, cfg.slm.head_dim, seq_lens)
    a = attend_bytes_coherent(cfg.llm.kv_heads, cfg.llm.head_dim, seq_lens, budgets)
    return {"slm_score": s, "attend_per_layer": a, "step": s + llm_layers * a}
