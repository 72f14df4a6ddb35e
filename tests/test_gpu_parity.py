"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle.

Bars: selection bit-exact except the 1e-6 boundary band,
counts exact; outputs row-normwise relative error <= 2e-3 with the oracle
evaluated on the GPU's verified sets.  Inputs are seeded synthetic, at sizes
the oracle finishes in seconds yet spanning several tiles/chunks and ragged
tails, plus sampled checks at BASELINE.json's full config-2 size.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

import smallkv_synth as synth
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2508_02751_b200 import build
    build.build()
    torch.cuda.set_device(0)


def _check(p, layers=None, logit_atol=2e-4):
    step, out_sel, outs = parity.run_gpu_step(p, layers=layers)
    sel = parity.oracle_select(p)
    rep = parity.compare_select(p, out_sel, sel, logit_atol=logit_atol)
    sg = parity.sel_from_gpu(p, out_sel, sel)
    errs = []
    for i, slot in enumerate(range(p.llm.num_layers) if layers is None else layers):
        e, _ = parity.compare_attend(p, slot, outs[i], sg)
        errs.append(e)
        assert e <= parity.OUT_TOL, f"layer slot {slot}: row-normwise err {e}"
    rep["max_out_err"] = max(errs) if errs else 0.0
    return rep, out_sel, outs


def _cfg(llm=(2, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=3, budget=(150, 60, 200)):
    return synth.small_config(llm=llm, slm=slm, seq_len=n, batch=B, budget=budget)


# ---------------------------------------------------------------- configs

def test_toy_config_parity():
    """BASELINE.json configs[0] at full size: 20% critical + 30% marginal."""
    p = synth.make_problem(synth.CONFIGS["toy"], seed=11).to("cuda")
    rep, _, _ = _check(p)
    print("toy", rep)


@pytest.mark.parametrize("page_size", [1, 16, 64])
@pytest.mark.parametrize("map_kind", ["coherent", "random"])
def test_small_parity_pages_maps(page_size, map_kind):
    """Several 1024-position chunks, ragged lengths, every page size."""
    cfg = _cfg(n=2600, B=3)
    p = synth.make_problem(cfg, seed=5, page_size=page_size, seq_lens=[2600, 1337, 65],
                           map_kind=map_kind).to("cuda")
    rep, _, _ = _check(p)
    print(page_size, map_kind, rep)


@pytest.mark.parametrize("dims", [
    ((1, 28, 4, 128), (2, 14, 2, 64)),   # qwen7b-shaped G=7, G_s=7
    ((1, 32, 8, 128), (1, 32, 8, 64)),   # llama-shaped G=4, G_s=4
    ((1, 40, 8, 128), (1, 12, 2, 128)),  # qwen14b-shaped G=5, d_s=128
    ((1, 64, 8, 128), (1, 14, 2, 64)),   # qwen72b-shaped G=8
    ((1, 4, 2, 64), (1, 2, 1, 64)),      # toy-shaped d=64
])
def test_shapes_parity(dims):
    llm, slm = dims
    cfg = _cfg(llm=llm, slm=slm, n=1100, B=2, budget=(110, 55, 110))
    p = synth.make_problem(cfg, seed=7, page_size=16, seq_lens=[1100, 700],
                           map_kind="random").to("cuda")
    rep, _, _ = _check(p)
    print(dims, rep)


# ---------------------------------------------------------------- special cases

def test_full_budget_is_dense_attention():
    """K'+R' = n, M = 0 => dense attention (pin P1 on the GPU)."""
    cfg = _cfg(n=1200, B=2, budget=(100000, 33, 0))
    p = synth.make_problem(cfg, seed=3, page_size=16, seq_lens=[1200, 513]).to("cuda")
    _check(p)


def test_marginal_only_and_empty():
    for budget in [(0, 0, 100000), (0, 0, 0), (0, 40, 0), (0, 0, 5)]:
        cfg = _cfg(n=900, B=2, budget=budget)
        p = synth.make_problem(cfg, seed=4, page_size=16, seq_lens=[900, 301]).to("cuda")
        rep, _, outs = _check(p)
        if budget == (0, 0, 0):
            assert all(torch.count_nonzero(o).item() == 0 for o in outs)


def test_clamp_short_sequences():
    """n below K+R+M and n = 1 (device clamp R5)."""
    cfg = _cfg(n=300, B=4, budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=8, page_size=16, seq_lens=[300, 1, 2, 61]).to("cuda")
    _check(p)


def test_zero_query_all_ties():
    """q' = 0: every logit ties; lower index wins (R3) — exact lists."""
    cfg = _cfg(n=1500, B=2)
    p = synth.make_problem(cfg, seed=9, page_size=16, seq_lens=[1500, 999])
    p = dataclasses.replace(p, slm_q=torch.zeros_like(p.slm_q)).to("cuda")
    rep, sel, _ = _check(p)
    crit, marg, cnt = sel.crit.cpu(), sel.marg.cpu(), sel.counts.cpu()
    for j in np.unique(p.head_map.cpu().numpy()):
        for b in range(p.batch):
            K, M = int(cnt[j, b, 0]), int(cnt[j, b, 1])
            assert crit[j, b, :K].tolist() == list(range(K))
            assert marg[j, b, :M].tolist() == list(range(K, K + M))


def test_duplicate_keys_exact_ties():
    """Duplicated K' rows give exactly equal logits; index tie-break decides."""
    cfg = _cfg(n=1024, B=1, budget=(100, 20, 100))
    p = synth.make_problem(cfg, seed=10, page_size=64, seq_lens=[1024])
    k = p.slm.k.clone()
    k[:, :, :, 1::2] = k[:, :, :, 0::2]      # rows 2i+1 := rows 2i in every page
    p = dataclasses.replace(p, slm=dataclasses.replace(p.slm, k=k)).to("cuda")
    _check(p)


@pytest.mark.parametrize("n", [4000, 8000, 12000, 14000, 20000])
def test_massive_ties_radix_fallback(n):
    """Two distinct K' rows (alternating by page): two distinct logits, so the
    boundary bins (and their sub-bins) hold thousands of equal keys and K2 takes
    the exact radix select + index tie-break.  n covers the K2 variants at
    B = 1: register rows (256 x 16, 512 x 16, 512 x 24), the long split
    (14000) and the cluster split (20000 > 16384 with < 1024 pairs)."""
    cfg = _cfg(n=n, B=1, budget=(n // 10, 20, n // 10))
    p = synth.make_problem(cfg, seed=21, page_size=256, seq_lens=[n])
    k = p.slm.k.clone()
    k[:, 0::2] = p.slm.k[:, :1, :, :1]        # even pages: page 0's first row
    k[:, 1::2] = p.slm.k[:, 1:2, :, :1]       # odd pages: page 1's first row
    p = dataclasses.replace(p, slm=dataclasses.replace(p.slm, k=k)).to("cuda")
    _check(p)


def test_extreme_logits():
    """Logits near ±80 (fp32 exp underflow): ranking on logits stays exact."""
    cfg = _cfg(n=800, B=1, budget=(80, 20, 100))
    p = synth.make_problem(cfg, seed=12, page_size=16, seq_lens=[800])
    p = dataclasses.replace(p, slm_q=(p.slm_q.float() * 12).to(torch.bfloat16)).to("cuda")
    _check(p, logit_atol=5e-3)


# ---------------------------------------------------------------- invariants

def test_deterministic_and_page_permutation_invariant():
    cfg = _cfg(n=2100, B=2)
    p = synth.make_problem(cfg, seed=13, page_size=16, seq_lens=[2100, 1500],
                           map_kind="random").to("cuda")
    _, s1, o1 = parity.run_gpu_step(p)
    l1 = [s1.crit.clone(), s1.marg.clone(), s1.marg_w.clone(), s1.lse.clone()]
    _, s2, o2 = parity.run_gpu_step(p)
    for a, b in zip(l1, [s2.crit, s2.marg, s2.marg_w, s2.lse]):
        assert torch.equal(a, b)
    for a, b in zip(o1, o2):
        assert torch.equal(a, b)
    # permute the LLM physical pages: same logical cache, different addresses
    pages = p.llm.k.shape[1]
    perm = torch.randperm(pages, generator=torch.Generator().manual_seed(3)).cuda()
    inv = torch.argsort(perm)
    k2 = p.llm.k[:, inv]
    v2 = p.llm.v[:, inv]
    bt2 = perm[p.llm.block_table.long()].to(torch.int32)
    p2 = dataclasses.replace(p, llm=dataclasses.replace(p.llm, k=k2.contiguous(),
                                                         v=v2.contiguous(), block_table=bt2))
    _, _, o3 = parity.run_gpu_step(p2)
    for a, b in zip(o1, o3):
        assert torch.equal(a, b)


def test_launch_chains_bit_identical():
    """The programmatic launch chains give the same bits: row_flags -> K1 -> K2 ->
    plan -> attend (default), no plan (attend stages its own lists), and K1 / K2
    in SLM-layer chunks with K2 on an auxiliary stream (overlap_select)."""
    from paper_2508_02751_b200 import smallkv
    cfg = _cfg(llm=(3, 8, 2, 128), slm=(5, 8, 2, 64), n=1700, B=3)
    p = synth.make_problem(cfg, seed=15, page_size=16, seq_lens=[1700, 333, 1024],
                           map_kind="random").to("cuda")
    runs = []
    for kw in ({}, {"use_plan": False}, {"overlap_select": True}):
        for _ in range(2):   # a second replay on the same buffers
            _, sel, outs = parity.run_gpu_step(p, step=smallkv.from_problem(p, **kw))
            runs.append(([sel.crit.clone(), sel.marg.clone(), sel.marg_w.clone(),
                          sel.lse.clone(), sel.counts.clone()], [o.clone() for o in outs]))
    ref_sel, ref_out = runs[0]
    for s_, o_ in runs[1:]:
        for a, b in zip(ref_sel, s_):
            assert torch.equal(a, b)
        for a, b in zip(ref_out, o_):
            assert torch.equal(a, b)


def test_batch_partition_invariant():
    """A sequence's result does not depend on its batch neighbours (P12)."""
    cfg = _cfg(n=1500, B=4)
    p = synth.make_problem(cfg, seed=14, page_size=16, seq_lens=[1500, 900, 1200, 30]).to("cuda")
    st_all, _, o_all = parity.run_gpu_step(p)
    for idx in ([0, 1], [2, 3]):
        sub = dataclasses.replace(
            p, seq_lens=p.seq_lens[idx].contiguous(), slm_q=p.slm_q[:, idx].contiguous(),
            llm_q=p.llm_q[:, idx].contiguous(),
            slm=dataclasses.replace(p.slm, block_table=p.slm.block_table[idx].contiguous()),
            llm=dataclasses.replace(p.llm, block_table=p.llm.block_table[idx].contiguous()),
            k_crit=p.k_crit[idx].contiguous(), n_recent=p.n_recent[idx].contiguous(),
            k_marg=p.k_marg[idx].contiguous(), max_seq_len=p.max_seq_len)
        st_sub, _, o_sub = parity.run_gpu_step(sub)
        same = parity.attend_split(st_all) == parity.attend_split(st_sub)
        for a, b in zip(o_all, o_sub):
            parity.assert_same_outputs(a[idx], b, same)


# ---------------------------------------------------------------- matching

def test_match_heads_vs_oracle():
    import oracle
    from paper_2508_02751_b200 import smallkv
    rng = np.random.default_rng(0)
    for w, k, n_llm, n_slm in [(150, 30, 784, 336), (200, 40, 96, 50), (100, 16, 20, 7)]:
        llm_F = rng.integers(0, 50, (n_llm, w)).astype(np.float32) / 7.0  # ties
        slm_F = rng.random((n_slm, w)).astype(np.float32)
        slm_F[: min(5, n_slm)] = llm_F[: min(5, n_slm)] * 3.0
        hm, jac = smallkv.match_heads(torch.from_numpy(llm_F).cuda(),
                                      torch.from_numpy(slm_F).cuda(), k)
        ohm, ojac = oracle.match_heads(llm_F.astype(np.float64), slm_F.astype(np.float64), k)
        assert np.array_equal(hm.cpu().numpy(), ohm)
        np.testing.assert_allclose(jac.cpu().numpy(), ojac, rtol=1e-6)


# ---------------------------------------------------------------- full size (config 2)

@pytest.mark.slow
def test_qwen7b_full_size_sampled():
    """BASELINE.json configs[1] at full size (n=4096, B=32, all SLM layers),
    two resident LLM layers; selection checked on sampled rows/sequences,
    outputs on every head of the sampled sequences."""
    cfg = synth.CONFIGS["qwen7b"]
    p = synth.make_problem(cfg, seed=1, device="cuda", llm_layers=[0, 27])
    step, sel_gpu, outs = parity.run_gpu_step(p)
    pc = p.to("cpu")
    rows = np.unique(pc.head_map.numpy())
    rng = np.random.default_rng(0)
    sample_rows = np.sort(rng.choice(rows, 16, replace=False)).astype(np.int32)
    slm_view, llm_view = parity.views(pc)
    sel = parity.oracle_select(pc, rows=sample_rows, slm_view=slm_view)
    sb = sorted(rng.choice(pc.batch, 6, replace=False).tolist())
    rep = parity.compare_select(pc, sel_gpu, sel, batch_idx=sb)
    # outputs for sampled sequences: oracle on all rows the layer uses
    used = np.unique(np.concatenate([pc.head_map.numpy()[l * cfg.llm.q_heads:(l + 1) * cfg.llm.q_heads]
                                     for l in (0, 27)])).astype(np.int32)
    sel_used = parity.oracle_select(pc, rows=used, slm_view=slm_view)
    parity.compare_select(pc, sel_gpu, sel_used, batch_idx=sb)
    sg = parity.sel_from_gpu(pc, sel_gpu, sel_used)
    for slot in range(2):
        e, _ = parity.compare_attend(pc, slot, outs[slot].cpu(), sg, llm_view=llm_view,
                                     heads=sb)
        assert e <= parity.OUT_TOL
    print("qwen7b sampled", rep)


def test_two_valued_logits_radix_fallback():
    """Logits taking two values: > 1024 positions share the boundary bin of the
    histogram path, forcing the radix fallback of K2 (ties by index)."""
    cfg = _cfg(n=3000, B=2, budget=(500, 100, 700))
    p = synth.make_problem(cfg, seed=15, page_size=16, seq_lens=[3000, 2500])
    k = p.slm.k.clone()
    k[..., 0::2, :] = k[0, 0, 0, 0]       # even rows of every page: one vector
    k[..., 1::2, :] = k[0, 0, 0, 1]       # odd rows: another
    p = dataclasses.replace(p, slm=dataclasses.replace(p.slm, k=k)).to("cuda")
    _check(p)


@pytest.mark.parametrize("n", [32000, 14000, 4000])
def test_dense_boundary_bin_refinement(n):
    """A few outlier logits stretch the value-linear histogram so that the
    boundary bin holds thousands of positions: K2 refines inside that bin
    (256 sub-bins) instead of falling back to the radix select.  n = 4000 runs
    the register-row variant (rows <= 4096 tokens), whose refinement re-reads
    the row from global memory."""
    cfg = _cfg(n=n, B=1, budget=(n // 10, n // 64, n // 10))
    p = synth.make_problem(cfg, seed=17, page_size=64, seq_lens=[n])
    k = p.slm.k.clone()
    k[:, :, :, 3] *= 40.0                 # one row per page: far outliers (both signs)
    p = dataclasses.replace(p, slm=dataclasses.replace(p.slm, k=k)).to("cuda")
    rep, _, _ = _check(p, logit_atol=2e-3)
    print("refinement", rep)


@pytest.mark.parametrize("n", [8000, 12000])
def test_register_split_radix_threshold(n):
    """Rows of 4097..12288 tokens take the 512-thread register split; a
    boundary bin of more than 48 pairs gets its exact threshold pair by a
    one-warp radix select instead of per-position rank counting.  Outliers
    (one row per page x3) squeeze the bulk into fewer of the 256 linear bins so
    that some boundary bin of some row is that long (checked on the GPU's own
    logits with the split's bin formula), and the split matches the oracle."""
    import numpy as np
    cfg = _cfg(n=n, B=2, budget=(n // 10, n // 64, n // 10))
    p = synth.make_problem(cfg, seed=19, page_size=64, seq_lens=[n, n - 777])
    k = p.slm.k.clone()
    k[:, :, :, 5] *= 3.0
    p = dataclasses.replace(p, slm=dataclasses.replace(p.slm, k=k)).to("cuda")
    rep, out_sel, _ = _check(p)
    logits = out_sel.logits.float().cpu().numpy()
    longest = 0
    for j in sorted(set(p.head_map.cpu().tolist())):   # the rows K1 scored
        for b in range(p.batch):
            nb = int(p.seq_lens[b])
            R = min(int(p.n_recent[b]), nb)
            N = nb - R
            K = min(int(p.k_crit[b]), N)
            M = min(int(p.k_marg[b]), N - K)
            v = logits[j, b, :N].astype(np.float32)
            if N == 0 or not v.max() > v.min():
                continue
            scale = np.float32(255.99) / (np.float32(v.max()) - np.float32(v.min()))
            bins = np.clip(((v - np.float32(v.min())) * scale).astype(np.int32), 0, 255)
            cnt = np.bincount(bins, minlength=256)[::-1]
            cum = np.cumsum(cnt)
            for r in (K, K + M):
                if r > 0:
                    longest = max(longest, int(cnt[np.searchsorted(cum, r)]))
    assert longest > 48, longest   # the radix-select branch ran for some row
    print("radix threshold", n, "longest boundary bin", longest, rep)


def _head_shard(p, g0, g1):
    from paper_2508_02751_b200 import dist as pdist
    L, H, Hkv = p.cfg.llm.layers, p.cfg.llm.q_heads, p.cfg.llm.kv_heads
    k, v, q, hm = pdist.slice_llm_kv_groups(p.llm.k, p.llm.v, p.llm_q, p.head_map, L, H, Hkv,
                                            g0, g1)
    G = H // Hkv
    dims = synth.ModelDims(L, (g1 - g0) * G, g1 - g0, p.cfg.llm.head_dim)
    cfg = dataclasses.replace(p.cfg, llm=dims)
    return dataclasses.replace(p, cfg=cfg, llm=dataclasses.replace(p.llm, k=k, v=v, dims=dims),
                               llm_q=q, head_map=hm)


def test_head_split_virtual_shards_bit_identical():
    """KV-head-group sharding (2 virtual ranks on one GPU): each shard's output
    slice equals the unsharded output bit for bit (partition invariance P12)."""
    cfg = _cfg(llm=(2, 8, 4, 128), slm=(2, 8, 2, 64), n=1800, B=2)
    p = synth.make_problem(cfg, seed=16, page_size=16, seq_lens=[1800, 1000],
                           map_kind="random").to("cuda")
    st_full, _, full = parity.run_gpu_step(p)
    for g0, g1 in [(0, 2), (2, 4)]:
        st_part, _, part = parity.run_gpu_step(_head_shard(p, g0, g1))
        same = parity.attend_split(st_full) == parity.attend_split(st_part)
        for a, b in zip(full, part):
            parity.assert_same_outputs(a[:, g0 * 2:g1 * 2], b, same)


def _full_size_sampled(cfg, *, budget=None, n_rows=6, n_seqs=2, seed=2, layers=(0, 1)):
    """Full BASELINE size on the GPU (all SLM layers, the given LLM layers
    resident); selection checked on sampled rows x sequences, outputs of the
    sampled sequences for every head of the resident layers."""
    p = synth.make_problem(cfg, seed=seed, device="cuda", llm_layers=list(layers),
                           budget=budget)
    step, sel_gpu, outs = parity.run_gpu_step(p)
    rng = np.random.default_rng(seed)
    sb = sorted(rng.choice(p.batch, n_seqs, replace=False).tolist())
    # only the sampled sequences go to the CPU: slice batch-indexed inputs
    sub = dataclasses.replace(
        p, seq_lens=p.seq_lens[sb].contiguous(), slm_q=p.slm_q[:, sb].contiguous(),
        llm_q=p.llm_q[:, sb].contiguous(),
        slm=dataclasses.replace(p.slm, block_table=p.slm.block_table[sb].contiguous()),
        llm=dataclasses.replace(p.llm, block_table=p.llm.block_table[sb].contiguous()),
        k_crit=p.k_crit[sb].contiguous(), n_recent=p.n_recent[sb].contiguous(),
        k_marg=p.k_marg[sb].contiguous()).to("cpu")

    class _SubSel:   # GPU selection outputs restricted to the sampled sequences
        pass
    gs = _SubSel()
    for name in ("logits", "lse", "crit", "marg", "marg_w", "counts"):
        setattr(gs, name, getattr(sel_gpu, name)[:, sb])
    H = cfg.llm.q_heads
    used = np.unique(np.concatenate(
        [sub.head_map.numpy()[l * H:(l + 1) * H] for l in layers])).astype(np.int32)
    sample = np.sort(rng.choice(used, min(n_rows, len(used)), replace=False)).astype(np.int32)
    slm_view, llm_view = parity.views(sub)
    rep = parity.compare_select(sub, gs, parity.oracle_select(sub, rows=sample,
                                                              slm_view=slm_view))
    sel_used = parity.oracle_select(sub, rows=used, slm_view=slm_view)
    parity.compare_select(sub, gs, sel_used)
    sg = parity.sel_from_gpu(sub, gs, sel_used)
    errs = []
    for slot in range(len(layers)):
        e, _ = parity.compare_attend(sub, slot, outs[slot][sb].cpu(), sg, llm_view=llm_view)
        errs.append(e)
        assert e <= parity.OUT_TOL
    rep["max_out_err"] = max(errs)
    return rep


@pytest.mark.slow
@pytest.mark.parametrize("tau", [0.05, 0.5])
def test_llama8b_full_size_sampled(tau):
    """BASELINE configs[2]: LLaMA-3.1-8B + 3.2-1B, n=32768, B=16, budget
    sweep end points (tau = 5% and 50%)."""
    cfg = synth.CONFIGS["llama8b"]
    print("llama8b", tau, _full_size_sampled(cfg, budget=synth.LLAMA8B_SWEEP[tau]))


@pytest.mark.slow
def test_qwen72b_full_size_sampled():
    """BASELINE configs[3]: Qwen2.5-72B + 0.5B, n=131072, B=8 (2 resident LLM
    layers of 80; layers 0 and 79 exercise both ends of the head map)."""
    cfg = synth.CONFIGS["qwen72b"]
    print("qwen72b", _full_size_sampled(cfg, layers=(0, 79), n_rows=4))


@pytest.mark.slow
def test_qwen14b_full_size_sampled():
    """BASELINE configs[4]: Qwen2.5-14B + 1.5B, start of the long generation
    (n=8193, B=64, d_s=128) and its end (n=16384, per-step tau budgets)."""
    cfg = synth.CONFIGS["qwen14b"]
    print("qwen14b n=8193", _full_size_sampled(cfg, n_seqs=3))
    cfg16 = dataclasses.replace(cfg, seq_len=16384, batch=16)
    print("qwen14b n=16384", _full_size_sampled(cfg16, budget=(1638, 819, 1638), n_seqs=2))


@pytest.mark.parametrize("n", [4096, 4097, 6000, 9000, 14000])
def test_select_row_storage_variants(n):
    """K2 keeps a row in registers (256 x 16 up to 4096 tokens, 512 x 16 up to
    8192, 512 x 24 up to 12288) or reads it from global memory (longer; f1
    rows: shared memory up to 8192): the same exact split
    from each, at the boundaries of the variants, with a ragged second
    sequence."""
    cfg = _cfg(n=n, B=2, budget=(n // 10, n // 20, n // 10))
    p = synth.make_problem(cfg, seed=23, page_size=16, seq_lens=[n, n // 3 + 1]).to("cuda")
    rep, _, _ = _check(p)
    print(n, rep)


@pytest.mark.parametrize("n0", [1500, 6000, 9000])
def test_f1_accumulated_score_multistep(n0):
    """Variant f1 over 4 decode steps (n grows by one each step): the GPU's
    running sums track the oracle's fp64 chain and the sets match within the
    A18 band (relative 1e-6 for sums > 1), outputs within 2e-3.  n0 covers the
    register / shared-memory / global K2 variants."""
    import oracle
    from paper_2508_02751_b200 import smallkv
    n1 = 900 if n0 == 1500 else n0 // 2
    cfg = _cfg(n=n0, B=2, budget=(120, 40, 160))
    p = synth.make_problem(cfg, seed=17, page_size=16, seq_lens=[n0, n1]).to("cuda")
    step = smallkv.from_problem(p)
    acc = torch.zeros_like(step.out.logits)
    pc = p.to("cpu")
    slm_view, llm_view = parity.views(pc)
    rows = oracle.image_rows(pc.head_map)
    oacc = np.zeros((len(rows), p.batch, p.max_seq_len), np.float64)
    for d in (3, 2, 1, 0):
        sl = torch.tensor([n0 - d, n1 - d], dtype=torch.int32)
        p.seq_lens.copy_(sl)
        sel_gpu = step.select(p.slm_q, acc=acc)
        torch.cuda.synchronize()
        sel = oracle.select_acc(pc.slm_q, slm_view, sl, rows, pc.k_crit, pc.n_recent,
                                pc.k_marg, p.max_crit, p.max_marg, p.max_seq_len, oacc)
    ga = acc.cpu().double().numpy()[rows]
    for b, n in enumerate([n0, n1]):
        np.testing.assert_allclose(ga[:, b, :n], oacc[:, b, :n], rtol=2e-5, atol=1e-7)
    # sets: ranked by the oracle's running sums
    pcs = dataclasses.replace(pc, seq_lens=sl)
    rep = parity.compare_select(pcs, sel_gpu, sel, rank_score=oacc)
    out = torch.empty(p.batch, cfg.llm.q_heads, cfg.llm.head_dim, device="cuda")
    step.attend(0, 0, p.llm_q[0], out)
    sg = parity.sel_from_gpu(pcs, sel_gpu, sel)
    e, _ = parity.compare_attend(pcs, 0, out, sg, llm_view=llm_view)
    assert e <= parity.OUT_TOL
    print("f1", rep, e)


# ---------------------------------------------------------------- variant f2 (R16)

def _check_group(p, layers=None):
    from paper_2508_02751_b200 import smallkv
    step = smallkv.from_problem(p, variant="f2")
    _, gout, outs = parity.run_gpu_step(p, step=step, layers=layers)
    sel = parity.oracle_select(p)
    reps = []
    for i, slot in enumerate(range(p.llm.num_layers) if layers is None else layers):
        reps.append(parity.compare_group(p, gout, sel, slot, out_gpu=outs[i]))
    return reps


@pytest.mark.parametrize("map_kind", ["random", "coherent"])
def test_f2_group_selection_parity(map_kind):
    """Variant f2: shared per-KV-group split of the summed proxy rows, per-head
    marginal weights; ragged lengths incl. n = 1, budgets over n (clamp)."""
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=4, budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=21, page_size=16, seq_lens=[1500, 731, 1, 200],
                           map_kind=map_kind).to("cuda")
    for rep in _check_group(p):
        print("f2", map_kind, rep)


@pytest.mark.parametrize("llm,slm", [((2, 28, 4, 128), (2, 14, 2, 64)),   # G = 7 (Qwen2.5-7B)
                                     ((2, 32, 8, 128), (2, 32, 8, 64)),   # G = 4
                                     ((1, 16, 16, 64), (1, 8, 8, 64))])   # G = 1, d = 64
def test_f2_shapes(llm, slm):
    cfg = _cfg(llm=llm, slm=slm, n=2100, B=2, budget=(210, 105, 210))
    p = synth.make_problem(cfg, seed=22, page_size=64, seq_lens=[2100, 1337]).to("cuda")
    for rep in _check_group(p):
        print("f2 shape", llm, rep)


def test_f2_qwen7b_dims():
    """f2 at config 2's model dims and context (n = 4096), 4 sequences."""
    cfg = synth.CONFIGS["qwen7b"]
    p = synth.make_problem(cfg, seed=23, batch=4, llm_layers=[0, 1]).to("cuda")
    for rep in _check_group(p):
        print("f2 qwen7b", rep)


# ---------------------------------------------------------------- variant f3 (R17)

@pytest.mark.parametrize("which,window", [("llm", (0, 150)), ("llm", (37, 123)),
                                          ("slm", (0, 200)), ("slm", (300, 200))])
def test_f3_prefill_scores_parity(which, window):
    """F (Eq. 1 column sums of the window's causal prefill rows) vs the fp64
    oracle; LLM d=128 G=4 / SLM d=64 G=2; windows at 0 and later (keep_last)."""
    import oracle
    from paper_2508_02751_b200 import smallkv
    start, length = window
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 4, 2, 64), n=start + length + 5, B=2)
    p = synth.make_problem(cfg, seed=31, page_size=16).to("cuda")
    cache = p.llm if which == "llm" else p.slm
    dims = cfg.llm if which == "llm" else cfg.slm
    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(cache.num_layers, length, dims.q_heads, dims.head_dim, device="cuda",
                    generator=g).to(torch.bfloat16)
    F = smallkv.prefill_scores(q, cache.k, cache.block_table, dims.q_heads, 1, start)
    view = oracle.CacheView(cache.k, None, cache.block_table, cache.num_pages, cache.page_size,
                            cache.num_layers, dims.q_heads, dims.kv_heads, dims.head_dim)
    ref = oracle.prefill_scores(q, view, 1, start, length)
    err = np.abs(F.cpu().double().numpy() - ref).max()
    print("f3", which, window, "max abs err", err, "max F", ref.max())
    assert err <= 1e-4 * max(1.0, ref.max())


def test_f3_head_matching_end_to_end():
    """Window -> LLM and SLM prefill F on the GPU -> K0 match_heads -> head map;
    equal to the oracle's match_heads on the GPU's F (Eq. 2-3), and the GPU F
    within tolerance of the oracle's F."""
    import oracle
    from paper_2508_02751_b200 import smallkv
    n = 420
    win = smallkv.match_window(n)
    assert win == oracle.match_window(n) == (220, 200)
    start, length = win
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 4, 2, 64), n=n, B=1)
    p = synth.make_problem(cfg, seed=32, page_size=16).to("cuda")
    g = torch.Generator(device="cuda").manual_seed(8)
    ql = torch.randn(2, length, 8, 128, device="cuda", generator=g).to(torch.bfloat16)
    qs = torch.randn(2, length, 4, 64, device="cuda", generator=g).to(torch.bfloat16)
    Fl = smallkv.prefill_scores(ql, p.llm.k, p.llm.block_table, 8, 0, start)
    Fs = smallkv.prefill_scores(qs, p.slm.k, p.slm.block_table, 4, 0, start)
    k_match = max(16, -(-length // 5))
    hm, jac = smallkv.match_heads(Fl, Fs, k_match)
    ohm, ojac = oracle.match_heads(Fl.cpu().double().numpy(), Fs.cpu().double().numpy(), k_match)
    assert np.array_equal(hm.cpu().numpy(), ohm)
    np.testing.assert_allclose(jac.cpu().numpy(), ojac, rtol=1e-6)
    lv = oracle.CacheView(p.llm.k, None, p.llm.block_table, p.llm.num_pages, p.llm.page_size,
                          2, 8, 2, 128)
    refl = oracle.prefill_scores(ql, lv, 0, start, length)
    assert np.abs(Fl.cpu().double().numpy() - refl).max() <= 1e-4 * max(1.0, refl.max())


# ---------------------------------------------------------------- variant f4 (R18)

def _tiered_step(p, variant="default", per_layer=False, host_layers=None):
    from paper_2508_02751_b200 import smallkv
    step = smallkv.from_problem(p, use_plan=False, variant=variant)
    src_k = p.llm.k if host_layers is None else p.llm.k[:host_layers]
    src_v = p.llm.v if host_layers is None else p.llm.v[:host_layers]
    host_k = torch.empty(src_k.shape, dtype=p.llm.k.dtype, pin_memory=True)
    host_v = torch.empty(src_v.shape, dtype=p.llm.v.dtype, pin_memory=True)
    host_k.copy_(src_k)
    host_v.copy_(src_v)
    G = p.cfg.llm.q_heads // p.cfg.llm.kv_heads
    cap = -(-(int(p.n_recent.max()) + G * (p.max_crit + p.max_marg)) // 4) * 4
    tier = smallkv.TieredKV(step, host_k, host_v, capacity=cap, use_plan=not per_layer,
                            per_layer=per_layer)
    return step, tier


def _run_both(p, step, tier, slm_q):
    """One decode step through the HBM pool and through the tiered pool."""
    step.select(slm_q)
    tier.update()
    outs = []
    for slot in range(p.llm.num_layers):
        layer = p.llm_layer_ids[slot]
        assert layer == slot   # f4: pool layer l holds LLM layer l
        ref = torch.empty(p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim, device="cuda")
        got = torch.empty_like(ref)
        step.attend(layer, slot, p.llm_q[slot], ref)
        tier.attend(layer, p.llm_q[slot], got)
        outs.append((ref, got))
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("variant,map_kind", [("default", "coherent"), ("default", "random"),
                                              ("f2", "random")])
def test_f4_tiered_pool_bitwise(variant, map_kind):
    """Host-resident pool + HBM hot pool: outputs bitwise equal to the
    HBM-resident path; a repeated step fetches nothing; a changed SLM query
    fetches only rows that were not resident."""
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=3, budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=41, page_size=16, seq_lens=[1500, 700, 1],
                           map_kind=map_kind).to("cuda")
    step, tier = _tiered_step(p, variant)
    for ref, got in _run_both(p, step, tier, p.slm_q):
        assert torch.equal(ref, got)
    f1, ov = tier.counters()
    assert ov == 0 and f1 > 0
    for ref, got in _run_both(p, step, tier, p.slm_q):      # same step again: all resident
        assert torch.equal(ref, got)
    f2_, _ = tier.counters()
    assert f2_ == f1, (f1, f2_)
    g = torch.Generator(device="cuda").manual_seed(3)
    q2 = (p.slm_q.float() + 0.5 * torch.randn(p.slm_q.shape, device="cuda", generator=g)).to(torch.bfloat16)
    for ref, got in _run_both(p, step, tier, q2):            # drifted selection: partial refetch
        assert torch.equal(ref, got)
    f3, ov = tier.counters()
    assert ov == 0 and f1 < f3 < 2 * f1, (f1, f3)
    print("f4", variant, map_kind, "rows fetched: first step", f1, "drifted step", f3 - f1)
    # and against the oracle on the GPU's own lists (default selection)
    if variant == "default":
        both = _run_both(p, step, tier, p.slm_q)   # back to the original query
        sel = parity.oracle_select(p)
        parity.compare_select(p, step.out, sel)
        sg = parity.sel_from_gpu(p, step.out, sel)
        for slot, (ref, got) in enumerate(both):
            e, _ = parity.compare_attend(p, slot, got, sg)
            assert e <= parity.OUT_TOL


def test_f4_long_context_and_rotated_host_pool():
    """f4 past the former 32768-token limit (bitmaps sized by max_seq_len, work
    lists in global memory): n = 40000 with a ragged second sequence, bitwise
    equal to the HBM-resident path and to the oracle; and a host pool of ONE
    layer slot serving both LLM layers (slot l mod 1), against the HBM path
    reading cache slot 0 for both."""
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 8, 2, 64), n=40000, B=2, budget=(4000, 2000, 4000))
    p = synth.make_problem(cfg, seed=45, page_size=64, seq_lens=[40000, 9001]).to("cuda")
    step, tier = _tiered_step(p)
    both = _run_both(p, step, tier, p.slm_q)
    for ref, got in both:
        assert torch.equal(ref, got)
    f1, ov = tier.counters()
    assert ov == 0 and f1 > 0
    sel = parity.oracle_select(p)
    parity.compare_select(p, step.out, sel)
    sg = parity.sel_from_gpu(p, step.out, sel)
    for slot, (ref, got) in enumerate(both):
        e, _ = parity.compare_attend(p, slot, got, sg)
        assert e <= parity.OUT_TOL
    # rotation: host slot l mod 1
    step1, tier1 = _tiered_step(p, host_layers=1)
    step1.select(p.slm_q)
    tier1.update()
    for layer in range(2):
        ref = torch.empty(p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim, device="cuda")
        got = torch.empty_like(ref)
        step1.attend(layer, 0, p.llm_q[layer], ref)
        tier1.attend(layer, p.llm_q[layer], got)
        torch.cuda.synchronize()
        assert torch.equal(ref, got), layer


def test_decode_graph_tier_per_layer_refresh():
    """DecodeGraph with the per-layer f4 refresh (each layer's tier update on a
    high-priority side stream, attend l waiting only for refresh l): outputs
    bitwise equal to the eager all-layer refresh, over a repeated step (nothing
    fetched) and a drifted one (only non-resident rows fetched)."""
    from paper_2508_02751_b200 import smallkv
    cfg = _cfg(llm=(3, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=3, budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=47, page_size=16, seq_lens=[1500, 700, 1]).to("cuda")
    step, tier = _tiered_step(p)
    g = torch.Generator(device="cuda").manual_seed(5)
    q2 = (p.slm_q.float() + 0.5 * torch.randn(p.slm_q.shape, device="cuda", generator=g)).to(torch.bfloat16)
    refs1 = [ref for ref, _ in _run_both(p, step, tier, p.slm_q)]
    refs2 = [ref for ref, _ in _run_both(p, step, tier, q2)]
    stepg, tierg = _tiered_step(p, per_layer=True)
    L = p.llm.num_layers
    shape = (p.batch, cfg.llm.q_heads, cfg.llm.head_dim)
    outs = torch.empty((L,) + shape, dtype=torch.float32, device="cuda")
    slm_q = p.slm_q.clone()
    plan = [(l, l, p.llm_q[l], outs[l]) for l in range(L)]
    graph = smallkv.DecodeGraph(stepg, slm_q, plan, tier=tierg)
    assert graph.kernels_per_step >= 2 * L
    for q, refs in ((p.slm_q, refs1), (p.slm_q, refs1), (q2, refs2)):
        slm_q.copy_(q)
        graph.replay()
        graph.stream.synchronize()
        if q is p.slm_q:
            f_before, _ = tierg.counters()
        for l in range(L):
            assert torch.equal(outs[l], refs[l]), l
    f_after, ov = tierg.counters()
    assert ov == 0 and f_after > f_before


def test_f3b_partitioned_slm_virtual_ranks_bit_identical():
    """f3b on one GPU with 2 virtual ranks: each scores / splits only its SLM row
    block (head-map subset), the blocks are exchanged (row copies standing in for
    the all-gather), and the attention over the exchanged selection is bitwise
    equal to the unsharded step."""
    from paper_2508_02751_b200 import dist as pdist, smallkv
    cfg = _cfg(llm=(2, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=3)
    p = synth.make_problem(cfg, seed=51, page_size=16, seq_lens=[1500, 800, 33],
                           map_kind="random").to("cuda")
    _, _, full = parity.run_gpu_step(p)
    n_slm = cfg.slm.layers * cfg.slm.q_heads
    steps = [smallkv.from_problem(p) for _ in range(2)]
    for r, st in enumerate(steps):
        j0, j1 = pdist.slm_row_block(n_slm, 2, r)
        st.select(p.slm_q, select_head_map=pdist.select_head_map(p.head_map, j0, j1), plan=False)
    target = steps[0]
    for name in pdist.SELECTION_FIELDS:
        j0, j1 = pdist.slm_row_block(n_slm, 2, 1)
        getattr(target.out, name)[j0:j1] = getattr(steps[1].out, name)[j0:j1]
    target.plan()
    for slot in range(p.llm.num_layers):
        out = torch.empty_like(full[slot])
        target.attend(p.llm_layer_ids[slot], slot, p.llm_q[slot], out, overlap_prologue=slot > 0)
        torch.cuda.synchronize()
        assert torch.equal(out, full[slot])


# ---------------------------------------------------------------- public API: graphs

@pytest.mark.parametrize("adjacent", [True, False])
def test_decode_graph_host_io_matches_device_run(adjacent):
    """DecodeGraph(host_io=...) (the e2e path of bench.py): q' and every layer's
    q copied in from pinned host memory, every layer's output read back inside
    the graph (pairs of layers in one copy when the buffers are adjacent, per
    layer otherwise; an odd layer count leaves a single last layer).  The host
    outputs equal the eager device run bit for bit, and the oracle check of the
    device run holds."""
    from paper_2508_02751_b200 import smallkv
    cfg = _cfg(llm=(3, 8, 2, 128), slm=(2, 8, 2, 64), n=1300, B=2, budget=(130, 50, 130))
    p = synth.make_problem(cfg, seed=31, page_size=16, seq_lens=[1300, 777]).to("cuda")
    L = p.llm.num_layers
    step, _, outs_ref = parity.run_gpu_step(p)
    shape = (p.batch, cfg.llm.q_heads, cfg.llm.head_dim)
    if adjacent:
        outs_all = torch.empty((L,) + shape, dtype=torch.float32, device="cuda")
        outs = [outs_all[l] for l in range(L)]
        h_out = torch.zeros((L,) + shape, dtype=torch.float32, pin_memory=True)
    else:
        outs = [torch.empty(shape, dtype=torch.float32, device="cuda") for _ in range(L)]
        h_out = [torch.zeros(shape, dtype=torch.float32, pin_memory=True) for _ in range(L)]
    h_slm_q = p.slm_q.cpu().pin_memory()
    h_q = [p.llm_q[l].cpu().pin_memory() for l in range(L)]
    q_dev = [torch.zeros_like(p.llm_q[l]) for l in range(L)]
    slm_q_dev = torch.zeros_like(p.slm_q)
    plan = [(p.llm_layer_ids[l], l, q_dev[l], outs[l]) for l in range(L)]
    g = smallkv.DecodeGraph(step, slm_q_dev, plan, host_io=(h_slm_q, h_q, h_out))
    for _ in range(2):
        g.replay()
    g.stream.synchronize()
    for l in range(L):
        assert torch.equal(h_out[l], outs_ref[l].cpu()), l
    rep, _, _ = _check(p)
    print("host_io", adjacent, rep)


def test_decode_graph_host_io_tiered():
    """DecodeGraph(host_io=..., tier=...) (bench.py --variant f4 e2e): select,
    the hot-pool refresh and the tiered attends with the host copies inside the
    graph; the host outputs equal the eager tiered step bit for bit and the
    HBM-resident step's outputs."""
    from paper_2508_02751_b200 import smallkv
    cfg = _cfg(llm=(3, 8, 2, 128), slm=(2, 8, 2, 64), n=1500, B=3, budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=43, page_size=16, seq_lens=[1500, 700, 1]).to("cuda")
    step, tier = _tiered_step(p)
    refs = [ref for ref, _ in _run_both(p, step, tier, p.slm_q)]
    L = p.llm.num_layers
    shape = (p.batch, cfg.llm.q_heads, cfg.llm.head_dim)
    outs_all = torch.empty((L,) + shape, dtype=torch.float32, device="cuda")
    h_out = torch.zeros((L,) + shape, dtype=torch.float32, pin_memory=True)
    h_slm_q = p.slm_q.cpu().pin_memory()
    h_q = [p.llm_q[l].cpu().pin_memory() for l in range(L)]
    q_dev = [torch.zeros_like(p.llm_q[l]) for l in range(L)]
    plan = [(l, l, q_dev[l], outs_all[l]) for l in range(L)]
    g = smallkv.DecodeGraph(step, torch.zeros_like(p.slm_q), plan, host_io=(h_slm_q, h_q, h_out),
                            tier=tier)
    for _ in range(2):
        g.replay()
    g.stream.synchronize()
    for l in range(L):
        assert torch.equal(h_out[l], refs[l].cpu()), l


@pytest.mark.parametrize("cta", ["512", "1024"])
def test_long_split_cta_sizes(cta):
    """The long split's CTA size is a launch-time knob (SMALLKV_LONG_CTA, read
    once per process; 256 by default): rerun the long-row cases — ties with the
    radix fallback, the sub-bin refinement, two ragged sequences — in a fresh
    process at 512 and 1024 threads per CTA."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sel = ("test_massive_ties_radix_fallback and 14000 or test_dense_boundary_bin_refinement and 14000"
           " or test_select_row_storage_variants and 14000")
    env = dict(os.environ, SMALLKV_LONG_CTA=cta)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout, r.stdout[-2000:]



def test_attend_stream_k_split():
    """Stream-K attend (SMALLKV_ATTEND_FLAT=1, read once per process): when the
    groups do not divide the SMs, #SMs CTAs take equal byte shares of all
    groups laid end to end (a CTA spans the tail of one group and the head of
    the next; a group's shares merge in share order through the workspace).
    Rerun in a fresh process the parity cases whose group counts trigger it —
    6 groups (3 x 2; 26 shares per group at most), 8 and 16 (the shape
    cases), 128 (config 2 at full size: 148 CTAs, a group spans 2 or 3) — plus
    per-sequence budget mixes, empty / marginal-only budgets and ragged
    lengths, against the fp64 oracle; per-KV-head shared selection (f2); and
    the tiered pool (f4) and the decode graph, bitwise against the
    HBM-resident / device runs of the same mode."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sel = ("test_small_parity_pages_maps or test_shapes_parity or test_full_budget_is_dense_attention"
           " or test_marginal_only_and_empty or test_clamp_short_sequences or test_extreme_logits"
           " or test_qwen7b_full_size_sampled or test_per_sequence_budgets"
           " or test_f4_tiered_pool_bitwise or test_f4_long_context or test_decode_graph"
           " or test_f2_group_selection_parity or test_f2_shapes")
    env = dict(os.environ, SMALLKV_ATTEND_FLAT="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        os.path.join(root, "tests", "test_gpu_corners.py")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]
