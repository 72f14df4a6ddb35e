"""Memory-safety checks of every launch chain (compute-sanitizer is closed on
this GPU pool, so these stand in for memcheck / initcheck; racecheck's role is
played by bitwise run-to-run determinism).

For each chain — the default row_flags -> K1 -> K2 -> plan -> attend x L with
the PDL overlap prologue, no plan, K1/K2 in SLM-layer chunks with K2 on an
auxiliary stream, variant f1 (accumulated scores), f2 (group selection), f4
(tiered pool, including a capacity overflow) and f3 (prefill scores + K0):
  * out-of-bounds WRITES: every output, workspace and plan buffer is a view
    inside a larger allocation whose guard bands (64 KiB each side) hold a
    byte pattern that must survive the calls;
  * reads of UNINITIALISED memory: the same buffers are filled with 0xFF
    bytes (NaN / -1) instead of zeros before the calls; the results must be
    bitwise identical to the zero-initialised run;
  * reads OUTSIDE the cache: physical pages no block table references and the
    rows past n_b of every sequence's last page hold NaN; the outputs must be
    finite and bitwise identical to a run on unpoisoned caches.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

import smallkv_synth as synth

pytestmark = pytest.mark.gpu

GUARD = 64 * 1024
PATTERN = 0xA5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2508_02751_b200 import build
    build.build()
    torch.cuda.set_device(0)


class Guarded:
    """Views of `like`-shaped tensors inside guard-banded byte allocations."""

    def __init__(self, fill: int):
        self.fill = fill
        self.allocs = []

    def make(self, shape, dtype):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        raw = torch.full((n + 2 * GUARD + 16,), PATTERN, dtype=torch.uint8, device="cuda")
        inner = raw[GUARD:GUARD + n]
        inner.fill_(self.fill)
        self.allocs.append(raw)
        return inner.view(dtype).view(shape)

    def check(self):
        torch.cuda.synchronize()
        for raw in self.allocs:
            assert bool((raw[:GUARD] == PATTERN).all()), "write below a buffer"
            assert bool((raw[-GUARD - 16:] == PATTERN).all()), "write past a buffer"


def guard_step(st, fill: int) -> Guarded:
    """Re-point a DecodeStep's outputs, workspaces and plan into guarded views."""
    from paper_2508_02751_b200 import smallkv
    g = Guarded(fill)
    o = st.out
    st.out = smallkv.SelectOut(*(g.make(t.shape, t.dtype) for t in
                                 (o.logits, o.lse, o.crit, o.marg, o.marg_w, o.counts)))
    if st.variant == "f2":
        go = st.gout
        st.gout = smallkv.SelectOut(
            g.make(go.logits.shape, go.logits.dtype), st.out.lse,
            *(g.make(t.shape, t.dtype) for t in (go.crit, go.marg, go.marg_w, go.counts)))
    # the select workspace carries no initialisation requirement: poisoned too;
    # the attend workspace is zeroed once by contract (include/smallkv.h)
    st.ws_select = g.make(st.ws_select.shape, torch.uint8)
    st.ws_attend = g.make(st.ws_attend.shape, torch.uint8).zero_()
    if st.plan_buf is not None:
        st.plan_buf = g.make(st.plan_buf.shape, torch.uint8)
    return g


def poison_cache(p):
    """NaN in every page no block table references and in the rows past n_b of
    each sequence's pages (bf16 0x7FC0)."""
    nan = torch.tensor(0x7FC0, dtype=torch.int16).view(torch.bfloat16).item()
    for cache in (p.slm, p.llm):
        used = torch.zeros(cache.num_pages, dtype=torch.bool, device="cuda")
        ps = cache.page_size
        for b, n in enumerate(p.seq_lens.tolist()):
            nb = -(-n // ps)
            pages = cache.block_table[b, :nb].long()
            used[pages] = True
            last = int(cache.block_table[b, nb - 1])
            tail = n - (nb - 1) * ps
            for t in (cache.k, cache.v):
                if t is not None and tail < ps:
                    t[:, last, :, tail:] = nan
            # pages of the block table past the sequence (if any) stay unreferenced
        for t in (cache.k, cache.v):
            if t is not None:
                t[:, ~used] = nan


def problem(spare=24, **kw):
    cfg = synth.small_config(llm=(2, 8, 2, 128), slm=(3, 8, 2, 64), seq_len=2100, batch=3,
                             budget=(150, 60, 200))
    return synth.make_problem(cfg, seed=91, page_size=16, seq_lens=[2100, 700, 37],
                              map_kind="random", spare_pages=spare, **kw).to("cuda")


def run_chain(p, chain: str, fill: int):
    """One decode step of `chain` with guarded buffers; returns (guards, results)."""
    from paper_2508_02751_b200 import smallkv
    kw = {"noplan": {"use_plan": False}, "aux": {"overlap_select": True},
          "f2": {"variant": "f2"}}.get(chain, {})
    st = smallkv.from_problem(p, **kw)
    g = guard_step(st, fill)
    res = []
    acc = None
    if chain == "f1":
        acc = g.make(st.out.logits.shape, torch.float32).zero_()
        st.select(p.slm_q, acc=acc)
        st.select(p.slm_q, acc=acc)
    else:
        st.select(p.slm_q)
    outs = []
    for i in range(p.llm.num_layers):
        out = g.make((p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim), torch.float32)
        st.attend(p.llm_layer_ids[i], i, p.llm_q[i], out, overlap_prologue=i > 0)
        outs.append(out)
    torch.cuda.synchronize()
    sel = st.gout if chain == "f2" else st.out
    rows = np.unique(p.head_map.cpu().numpy()) if chain != "f2" else \
        np.arange(p.cfg.llm.layers * p.cfg.llm.kv_heads)
    cnt = sel.counts.cpu()
    for r in rows:
        for b in range(p.batch):
            K, M = int(cnt[r, b, 0]), int(cnt[r, b, 1])
            res += [sel.crit[r, b, :K].cpu(), sel.marg[r, b, :M].cpu(),
                    sel.marg_w[r, b, :M].cpu()]
    res += [sel.counts[rows].cpu()] + [o.cpu() for o in outs]
    if acc is not None:
        res.append(acc[rows].cpu())
    return g, res


@pytest.mark.parametrize("chain", ["default", "noplan", "aux", "f1", "f2"])
def test_guards_poison_and_nan_pages(chain):
    p = problem()
    g0, clean = run_chain(p, chain, 0x00)
    g0.check()
    g1, dirty = run_chain(p, chain, 0xFF)          # uninitialised-read check
    g1.check()
    for a, b in zip(clean, dirty):
        assert torch.equal(a, b), chain
    pp = problem()
    poison_cache(pp)
    g2, nanrun = run_chain(pp, chain, 0xFF)        # out-of-cache read check
    g2.check()
    for a, b in zip(clean, nanrun):
        assert torch.equal(a, b), chain
    for o in nanrun[-(p.llm.num_layers + (1 if chain == "f1" else 0)):]:
        assert torch.isfinite(o).all()


def test_guards_tiered_pool_and_overflow():
    """f4: guarded hot pools / state; a capacity below the list size leaves the
    group's outputs NaN and touches nothing outside the buffers."""
    from paper_2508_02751_b200 import smallkv
    p = problem()
    poison_cache(p)
    for cap in (None, 64):
        st = smallkv.from_problem(p, use_plan=False)
        g = guard_step(st, 0xFF)
        hk = torch.empty(p.llm.k.shape, dtype=p.llm.k.dtype, pin_memory=True)
        hv = torch.empty(p.llm.v.shape, dtype=p.llm.v.dtype, pin_memory=True)
        hk.copy_(p.llm.k)
        hv.copy_(p.llm.v)
        G = p.cfg.llm.q_heads // p.cfg.llm.kv_heads
        c = cap or -(-(int(p.n_recent.max()) + G * (p.max_crit + p.max_marg)) // 4) * 4
        tier = smallkv.TieredKV(st, hk, hv, capacity=c)
        tier.hot_k = g.make(tier.hot_k.shape, torch.bfloat16)
        tier.hot_v = g.make(tier.hot_v.shape, torch.bfloat16)
        tier.state = g.make(tier.state.shape, torch.uint8)
        tier.reset()
        if tier.plan_buf is not None:
            tier.plan_buf = g.make(tier.plan_buf.shape, torch.uint8)
        st.select(p.slm_q)
        tier.update()
        outs = []
        for i in range(p.llm.num_layers):
            out = g.make((p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim), torch.float32)
            tier.attend(i, p.llm_q[i], out, overlap_prologue=i > 0)
            outs.append(out)
        g.check()
        if cap is None:
            ref = []
            for i in range(p.llm.num_layers):
                o = torch.empty_like(outs[i])
                st.attend(i, i, p.llm_q[i], o)
                ref.append(o)
            torch.cuda.synchronize()
            for a, b in zip(outs, ref):
                assert torch.equal(a, b) and torch.isfinite(a).all()
        else:
            assert tier.counters()[1] > 0
            # sequences 0, 1 (lists of >= 410 entries) overflow the 64 slots: NaN;
            # sequence 2 (n = 37) fits and is computed
            for o in outs:
                assert torch.isnan(o[:2]).all() and torch.isfinite(o[2]).all()


def test_guards_prefill_and_match():
    """f3 prefill scores and K0 match_heads into guarded outputs (the ABI
    allocates nothing; the Python wrappers' outputs are re-pointed here)."""
    import ctypes
    from paper_2508_02751_b200 import smallkv
    p = problem()
    poison_cache(p)
    lib = smallkv.load()
    gd = Guarded(0xFF)
    gq = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(p.llm.num_layers, 150, 8, 128, device="cuda", generator=gq).to(torch.bfloat16)
    cache = smallkv.make_cache(p.llm.k, None, p.llm.block_table, 8)
    F = gd.make((p.llm.num_layers * 8, 150), torch.float32)
    rc = lib.smallkv_prefill_scores(q.data_ptr(), ctypes.byref(cache), 0, 100, 150, F.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    Fr = smallkv.prefill_scores(q, p.llm.k, p.llm.block_table, 8, 0, 100)
    torch.cuda.synchronize()
    assert torch.equal(F, Fr) and torch.isfinite(F).all()
    slm_F = torch.rand(24, 150, device="cuda", generator=gq)
    hm = gd.make((F.shape[0],), torch.int32)
    jac = gd.make((F.shape[0],), torch.float32)
    wsb = lib.smallkv_match_heads_workspace_size(F.shape[0], 24)
    ws = gd.make((max(wsb, 1),), torch.uint8)
    rc = lib.smallkv_match_heads(F.data_ptr(), F.shape[0], slm_F.data_ptr(), 24, 150, 30,
                                 hm.data_ptr(), jac.data_ptr(), ws.data_ptr(), ws.numel(),
                                 torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    hm2, jac2 = smallkv.match_heads(F, slm_F, 30)
    gd.check()
    assert torch.equal(hm, hm2) and torch.equal(jac, jac2)
