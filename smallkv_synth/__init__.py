"""Seeded synthetic decode inputs for SmallKV (shared by tests, bench and smoke).

This module holds NONE of the method's arithmetic: it only draws caches,
queries, page tables, head maps and integer budgets.  Both the CUDA path and
the CPU oracle consume what it produces; neither is imported here.

Recipe:
  * per sequence b a base salience z_b[v] ~ N(0, sigma_b^2), sigma_b in
    [0.9, 1.0], +3.8 on a 2% "heavy hitter" subset and +6 on the sink v=0 —
    calibrated to the sparsity shape of Fig. 2 (top-5% mass ≈ 7x the
    5-10% band);
  * LLM kv-group (layer, g) salience = z_b + N(0, 0.3^2); SLM kv-group
    salience = z_b + N(0, 0.4^2) (the SLM/LLM attention similarity of
    Insight 1, matched cosine ≈ 0.95);
  * K_v = xi_v + sqrt(d) * z_v * u_g with xi ~ N(0, I) and u_g a random unit
    direction per (layer, kv-group); group queries q_h = u_g + (0.3/sqrt(d)) eta_h
    (GQA heads of a group correlated), so q·K/sqrt(d) ≈ z + small noise;
  * V ~ N(0, 1); all tensors bf16;
  * paged HND pools [layer][page][kv_head][page_size][head_dim]; each
    model's block table is a seeded random permutation of its physical pages
    (no accidental contiguity); tokens past n_b in a page are never read.
  * head maps: "coherent" — every q-head of LLM group (layer, g) maps to one
    SLM q-head, spread round-robin over ALL SLM kv-heads so the full SLM K
    cache is referenced; "random" — each LLM head independently uniform over
    all SLM heads (stress case for per-head unions).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional, Sequence, Tuple

import torch

SEED_BASE = 250802751


@dataclasses.dataclass(frozen=True)
class ModelDims:
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    llm: ModelDims
    slm: ModelDims
    seq_len: int
    batch: int
    # explicit integer budgets (K critical, R recent, M marginal); the tau
    # they came from is recorded in `tau` (P:235 2:1:2 split, R6)
    budget: Tuple[int, int, int]
    tau: Optional[float]
    description: str


# BASELINE.json configs[0..4].  Budgets are written out as integers; for the
# tau presets they equal (floor(tau n/2), floor(tau n/4), floor(tau n/2)).
CONFIGS: Dict[str, Config] = {
    "toy": Config("toy", ModelDims(1, 4, 2, 64), ModelDims(1, 2, 1, 64), 512, 1,
                  (102, 0, 153), None,
                  "1 layer, LLM 4q/2kv d64, SLM 2q/1kv d64, ctx 512, batch 1, "
                  "20% critical + 30% marginal"),
    "qwen7b": Config("qwen7b", ModelDims(28, 28, 4, 128), ModelDims(24, 14, 2, 64), 4096, 32,
                     (409, 204, 409), 0.2,
                     "Qwen2.5-7B (28q/4kv d128) + Qwen2.5-0.5B (14q/2kv d64), ctx 4K, batch 32"),
    "llama8b": Config("llama8b", ModelDims(32, 32, 8, 128), ModelDims(16, 32, 8, 64), 32768, 16,
                      (3276, 1638, 3276), 0.2,
                      "LLaMA-3.1-8B + LLaMA-3.2-1B, ctx 32K, batch 16 (tau sweep 5-50%)"),
    "qwen72b": Config("qwen72b", ModelDims(80, 64, 8, 128), ModelDims(24, 14, 2, 64), 131072, 8,
                      (13107, 6553, 13107), 0.2,
                      "Qwen2.5-72B (64q/8kv) + Qwen2.5-0.5B, ctx 128K, batch 8"),
    "qwen14b": Config("qwen14b", ModelDims(48, 40, 8, 128), ModelDims(28, 12, 2, 128), 8193, 64,
                      (819, 409, 819), 0.2,
                      "Qwen2.5-14B + Qwen2.5-1.5B, 8K prompt + 8K decode, batch 64"),
}

# config 3's budget sweep, tau -> (K, R, M) at n = 32768
LLAMA8B_SWEEP = {0.05: (819, 409, 819), 0.1: (1638, 819, 1638), 0.2: (3276, 1638, 3276),
                 0.3: (4915, 2457, 4915), 0.4: (6553, 3276, 6553), 0.5: (8192, 4096, 8192)}


@dataclasses.dataclass
class PagedCache:
    k: torch.Tensor                 # bf16 [layers][pages][kv][page_size][d]
    v: Optional[torch.Tensor]       # same or None (SLM)
    block_table: torch.Tensor       # int32 [B][max_blocks]
    page_size: int
    dims: ModelDims

    @property
    def num_pages(self) -> int:
        return int(self.k.shape[1])

    @property
    def num_layers(self) -> int:
        return int(self.k.shape[0])


@dataclasses.dataclass
class Problem:
    cfg: Config
    seq_lens: torch.Tensor          # int32 [B]
    max_seq_len: int
    slm_q: torch.Tensor             # bf16 [l][B][H_s][d_s]
    slm: PagedCache
    llm_q: torch.Tensor             # bf16 [n_llm_q_layers][B][H][d] (one per resident layer)
    llm: PagedCache                 # layers = resident LLM layers
    llm_layer_ids: Sequence[int]    # logical LLM layer of each resident slot
    head_map: torch.Tensor          # int32 [L*H] -> flat SLM head
    k_crit: torch.Tensor            # int32 [B]
    n_recent: torch.Tensor
    k_marg: torch.Tensor
    max_crit: int
    max_marg: int

    @property
    def batch(self) -> int:
        return int(self.seq_lens.shape[0])

    def to(self, device) -> "Problem":
        def mv(x):
            return x.to(device) if isinstance(x, torch.Tensor) else x
        slm = dataclasses.replace(self.slm, k=mv(self.slm.k), v=mv(self.slm.v),
                                  block_table=mv(self.slm.block_table))
        llm = dataclasses.replace(self.llm, k=mv(self.llm.k), v=mv(self.llm.v),
                                  block_table=mv(self.llm.block_table))
        return dataclasses.replace(self, seq_lens=mv(self.seq_lens), slm_q=mv(self.slm_q),
                                   slm=slm, llm_q=mv(self.llm_q), llm=llm,
                                   head_map=mv(self.head_map), k_crit=mv(self.k_crit),
                                   n_recent=mv(self.n_recent), k_marg=mv(self.k_marg))


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def head_map_coherent(llm: ModelDims, slm: ModelDims) -> torch.Tensor:
    """Group-coherent map covering every SLM kv-head (see module docstring)."""
    G = llm.q_heads // llm.kv_heads
    G_s = slm.q_heads // slm.kv_heads
    n_slm_kv = slm.layers * slm.kv_heads
    out = torch.empty(llm.layers * llm.q_heads, dtype=torch.int32)
    for layer in range(llm.layers):
        for g in range(llm.kv_heads):
            t = layer * llm.kv_heads + g
            kv_flat = t % n_slm_kv
            s_layer, s_kv = divmod(kv_flat, slm.kv_heads)
            s_q = (t // n_slm_kv) % G_s
            j = s_layer * slm.q_heads + s_kv * G_s + s_q
            out[layer * llm.q_heads + g * G: layer * llm.q_heads + (g + 1) * G] = j
    return out


def head_map_random(llm: ModelDims, slm: ModelDims, seed: int) -> torch.Tensor:
    g = _gen(seed, "cpu")
    return torch.randint(0, slm.layers * slm.q_heads, (llm.layers * llm.q_heads,),
                         generator=g, dtype=torch.int64).to(torch.int32)


def _base_salience(B: int, n_max: int, g: torch.Generator, device) -> torch.Tensor:
    sigma = 0.9 + 0.1 * torch.rand(B, 1, generator=g, device=device)
    z = torch.randn(B, n_max, generator=g, device=device) * sigma
    heavy = torch.rand(B, n_max, generator=g, device=device) < 0.02
    z = z + 3.8 * heavy.float()
    z[:, 0] += 6.0
    return z


def _fill_pool(pool_layer: torch.Tensor, block_table: torch.Tensor, z: torch.Tensor,
               u: torch.Tensor, page_size: int, noise_sigma: float,
               g: torch.Generator, device):
    """pool_layer: [pages][kv][ps][d] (written). z: [B][n_pad] base salience,
    u: [kv][d] unit directions.  K rows = xi + sqrt(d) * (z + noise) * u."""
    B, n_pad = z.shape
    kv, d = u.shape
    nb = n_pad // page_size
    zg = z[:, None, :] + noise_sigma * torch.randn(B, kv, n_pad, generator=g, device=device)
    xi = torch.randn(B, kv, n_pad, d, generator=g, device=device)
    logical = xi + math.sqrt(d) * zg[..., None] * u[None, :, None, :]
    # [B][kv][nb][ps][d] -> [B][nb][kv][ps][d]
    logical = logical.view(B, kv, nb, page_size, d).permute(0, 2, 1, 3, 4)
    pool_layer[block_table[:, :nb].reshape(-1).long()] = (
        logical.reshape(B * nb, kv, page_size, d).to(torch.bfloat16))


def _unit(rows: int, d: int, g: torch.Generator, device) -> torch.Tensor:
    u = torch.randn(rows, d, generator=g, device=device)
    return u / u.norm(dim=-1, keepdim=True)


def make_problem(cfg: Config, *, seed: int = 0, device="cpu", page_size: int = 64,
                 seq_lens: Optional[Sequence[int]] = None, batch: Optional[int] = None,
                 llm_layers: Optional[Sequence[int]] = None, map_kind: str = "coherent",
                 budget: Optional[Tuple[int, int, int]] = None,
                 budgets_per_seq: Optional[Sequence[Tuple[int, int, int]]] = None,
                 spare_pages: int = 0) -> Problem:
    """Draw one decode step's inputs for `cfg`.

    seq_lens   per-sequence n_b (default cfg.seq_len for all); ragged allowed.
    batch      override cfg.batch (e.g. a per-rank shard).
    llm_layers logical LLM layers whose K/V/q are materialised (default all);
               the LLM pool holds exactly these, in order (layer rotation).
    """
    device = torch.device(device)
    B = batch if batch is not None else cfg.batch
    if seq_lens is None:
        seq_lens = [cfg.seq_len] * B
    assert len(seq_lens) == B
    n_max = max(seq_lens)
    nb = (n_max + page_size - 1) // page_size
    n_pad = nb * page_size
    g = _gen(SEED_BASE + 1000 * seed, device)
    gc = _gen(SEED_BASE + 1000 * seed + 7, "cpu")
    if llm_layers is None:
        llm_layers = list(range(cfg.llm.layers))

    z = _base_salience(B, n_pad, g, device)

    def paged(dims: ModelDims, n_layers_res: int, with_v: bool, noise: float,
              layer_ids: Sequence[int]):
        pages = B * nb + spare_pages
        perm = torch.randperm(pages, generator=gc)[: B * nb].view(B, nb).to(torch.int32)
        k = torch.zeros(n_layers_res, pages, dims.kv_heads, page_size, dims.head_dim,
                        dtype=torch.bfloat16, device=device)
        v = torch.zeros_like(k) if with_v else None
        us = []
        bt = perm.to(device)
        for slot, _layer in enumerate(layer_ids):
            u = _unit(dims.kv_heads, dims.head_dim, g, device)
            us.append(u)
            _fill_pool(k[slot], bt, z, u, page_size, noise, g, device)
            if with_v:
                vv = torch.randn(B * nb, dims.kv_heads, page_size, dims.head_dim,
                                 generator=g, device=device)
                v[slot][bt.reshape(-1).long()] = vv.to(torch.bfloat16)
        return PagedCache(k, v, bt, page_size, dims), us

    def queries(dims: ModelDims, us) -> torch.Tensor:
        G = dims.q_heads // dims.kv_heads
        qs = []
        for u in us:
            uq = u.repeat_interleave(G, dim=0)  # [H][d]
            eta = torch.randn(B, dims.q_heads, dims.head_dim, generator=g, device=device)
            qs.append(uq[None] + (0.3 / math.sqrt(dims.head_dim)) * eta)
        return torch.stack(qs).to(torch.bfloat16)

    slm_cache, slm_us = paged(cfg.slm, cfg.slm.layers, False, 0.4, list(range(cfg.slm.layers)))
    slm_q = queries(cfg.slm, slm_us)
    llm_cache, llm_us = paged(cfg.llm, len(llm_layers), True, 0.3, llm_layers)
    llm_q = queries(cfg.llm, llm_us)

    if map_kind == "coherent":
        hm = head_map_coherent(cfg.llm, cfg.slm)
    elif map_kind == "random":
        hm = head_map_random(cfg.llm, cfg.slm, SEED_BASE + 1000 * seed + 13)
    else:
        raise ValueError(map_kind)

    if budgets_per_seq is None:
        bud = budget if budget is not None else cfg.budget
        budgets_per_seq = [bud] * B
    kc = torch.tensor([x[0] for x in budgets_per_seq], dtype=torch.int32)
    nr = torch.tensor([x[1] for x in budgets_per_seq], dtype=torch.int32)
    km = torch.tensor([x[2] for x in budgets_per_seq], dtype=torch.int32)
    return Problem(cfg=cfg, seq_lens=torch.tensor(list(seq_lens), dtype=torch.int32).to(device),
                   max_seq_len=int(n_max), slm_q=slm_q, slm=slm_cache,
                   llm_q=llm_q, llm=llm_cache,
                   llm_layer_ids=list(llm_layers), head_map=hm.to(device),
                   k_crit=kc.to(device), n_recent=nr.to(device), k_marg=km.to(device),
                   max_crit=max(1, int(kc.max())), max_marg=max(1, int(km.max())))


def small_config(name: str = "small", *, llm=(2, 8, 2, 128), slm=(2, 4, 1, 64),
                 seq_len: int = 1000, batch: int = 3,
                 budget=(100, 50, 120)) -> Config:
    """Parity-sized config spanning several tiles with a ragged tail."""
    return Config(name, ModelDims(*llm), ModelDims(*slm), seq_len, batch, tuple(budget), None,
                  "parity-sized synthetic config")
