"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each test names the pin of DESIGN.md §5 (P1..P15) and the passage it follows.
None of them re-types the oracle's formula: they use SPEC/PAPER worked values,
library routines (torch SDPA / softmax / matmul, Python sorted), closed forms,
invariants or brute force on tiny inputs.
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
import random

import numpy as np
import pytest
import torch

import smallkv_synth as synth
from tests.helpers import brute_split, dense_rows, sdpa_fp64

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _views(oracle, p):
    slm = oracle.CacheView(p.slm.k, None, p.slm.block_table, p.slm.num_pages, p.slm.page_size,
                           p.slm.num_layers, p.cfg.slm.q_heads, p.cfg.slm.kv_heads,
                           p.cfg.slm.head_dim)
    llm = oracle.CacheView(p.llm.k, p.llm.v, p.llm.block_table, p.llm.num_pages,
                           p.llm.page_size, p.llm.num_layers, p.cfg.llm.q_heads,
                           p.cfg.llm.kv_heads, p.cfg.llm.head_dim)
    return slm, llm


def _run(oracle, p, layer_slot=0):
    slm, llm = _views(oracle, p)
    rows = oracle.image_rows(p.head_map)
    sel = oracle.select(p.slm_q, slm, p.seq_lens, rows, p.k_crit, p.n_recent, p.k_marg,
                        p.max_crit, p.max_marg, p.max_seq_len)
    layer = p.llm_layer_ids[layer_slot]
    out, wsum = oracle.attend(layer, layer_slot, p.llm_q[layer_slot], llm, p.seq_lens,
                              p.head_map, sel, p.cfg.slm.layers * p.cfg.slm.q_heads)
    return sel, out, wsum


def _small(seq_lens=(150, 97, 1), budget=(30, 10, 40), page_size=16, map_kind="random", seed=1):
    cfg = synth.small_config(llm=(2, 8, 2, 64), slm=(2, 4, 2, 64), seq_len=max(seq_lens),
                             batch=len(seq_lens), budget=budget)
    return synth.make_problem(cfg, seed=seed, page_size=page_size, seq_lens=list(seq_lens),
                              map_kind=map_kind)


def _slm_softmax(p, j, b):
    """SLM row of flat head j via torch softmax (fp64) on de-paged K'."""
    H_s = p.cfg.slm.q_heads
    G_s = H_s // p.cfg.slm.kv_heads
    layer, head = divmod(int(j), H_s)
    n = int(p.seq_lens[b])
    K = dense_rows(p.slm, layer, b, n, head // G_s, "k")
    q = p.slm_q[layer, b, head].double()
    s = (K @ q) / math.sqrt(p.cfg.slm.head_dim)
    return s, torch.softmax(s, dim=0)


# --------------------------------------------------------------------------- SPEC worked values

def test_spec_column_sums(oracle_mod):
    g = GOLDEN["column_sums_uniform_causal_n3"]
    F = oracle_mod.accumulate_scores(np.array(g["A"]))
    np.testing.assert_allclose(F, g["F"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("case", GOLDEN["topk"])
def test_spec_topk(oracle_mod, case):
    m = oracle_mod.topk_mask(case["scores"], case["k"])
    assert sorted(np.nonzero(m)[0].tolist()) == case["top"]


def test_spec_jaccard_via_match(oracle_mod):
    g = GOLDEN["jaccard"]
    w = 6
    fa = np.zeros(w); fa[g["a"]] = [3, 2, 1]
    fb = np.zeros(w); fb[g["b"]] = [3, 2, 1]
    hm, jac = oracle_mod.match_heads(fa[None], fb[None], 3)
    assert hm[0] == 0 and jac[0] == pytest.approx(g["value"], abs=1e-15)


def test_spec_evict_n4(oracle_mod):
    g = GOLDEN["evict_n4"]
    crit, marg, recent, counts = oracle_mod.split(g["scores"], g["critical"], g["recent"],
                                                  g["marginal"])
    e = g["expect"]
    assert crit.tolist() == e["critical"]
    assert marg.tolist() == e["marginal"]
    assert recent.tolist() == e["recent"]
    evicted = sorted(set(range(4)) - set(crit) - set(marg) - set(recent))
    assert evicted == e["evicted"]


# --------------------------------------------------------------------------- P5 brute force

def test_P5_split_bruteforce_1000():
    """>=1000 random instances, discrete scores to force ties (R3)."""
    import oracle
    rng = random.Random(7)
    for _ in range(1200):
        n = rng.randint(1, 64)
        levels = rng.choice([2, 3, 5, 1000])
        score = [rng.randint(0, levels) / levels for _ in range(n)]
        K, R, M = (rng.randint(0, n + 3) for _ in range(3))
        crit, marg, recent, counts = oracle.split(score, K, R, M)
        bc, bm, br, be = brute_split(score, K, R, M)
        assert crit.tolist() == bc and marg.tolist() == bm and recent.tolist() == br


def test_P6_zero_query_all_ties(oracle_mod):
    """q' = 0 => every a' equal => C = first K' of [0, n-R'), M = next M' (R3)."""
    p = _small(seq_lens=(120, 33), budget=(20, 7, 25))
    p = dataclasses.replace(p, slm_q=torch.zeros_like(p.slm_q))
    sel, _, _ = _run(oracle_mod, p)
    for r in range(len(sel["rows"])):
        for b in range(p.batch):
            n = int(p.seq_lens[b])
            Kc, Mc, Rc = sel["counts"][r, b]
            assert Rc == min(7, n)
            assert sel["crit"][r, b, :Kc].tolist() == list(range(Kc))
            assert sel["marg"][r, b, :Mc].tolist() == list(range(Kc, Kc + Mc))
            np.testing.assert_allclose(sel["a"][r, b, :n], 1.0 / n, rtol=1e-14)


# --------------------------------------------------------------------------- SLM rows

def test_slm_rows_vs_torch_softmax(oracle_mod):
    """a' = softmax(q'K'^T/sqrt(d_s)) via torch on de-paged K'; P7 sum = 1."""
    p = _small()
    sel, _, _ = _run(oracle_mod, p)
    for r, j in enumerate(sel["rows"]):
        for b in range(p.batch):
            n = int(p.seq_lens[b])
            s, a = _slm_softmax(p, j, b)
            np.testing.assert_allclose(sel["s"][r, b, :n], s.numpy(), rtol=1e-13, atol=1e-13)
            np.testing.assert_allclose(sel["a"][r, b, :n], a.numpy(), rtol=1e-12, atol=1e-15)
            assert abs(sel["a"][r, b, :n].sum() - 1.0) < 1e-12
            m, lse = sel["stats"][r, b]
            assert m == pytest.approx(float(s.max()), abs=1e-13)
            assert lse == pytest.approx(float(torch.logsumexp(s, 0)), abs=1e-12)


def test_P8_partition_and_bruteforce_sets(oracle_mod):
    """Sets disjoint, covering [0,n), sizes = clamp (R5); equal to a full sort of
    torch's softmax row (P5 on real rows)."""
    p = _small(seq_lens=(150, 40, 1, 7), budget=(30, 10, 40))
    sel, _, _ = _run(oracle_mod, p)
    for r, j in enumerate(sel["rows"]):
        for b in range(p.batch):
            n = int(p.seq_lens[b])
            Kc, Mc, Rc = (int(x) for x in sel["counts"][r, b])
            assert Rc == min(10, n) and Kc == min(30, n - Rc) and Mc == min(40, n - Rc - Kc)
            crit = sel["crit"][r, b, :Kc].tolist()
            marg = sel["marg"][r, b, :Mc].tolist()
            _, a = _slm_softmax(p, j, b)
            bc, bm, br, be = brute_split(a.tolist(), 30, 10, 40)
            assert crit == bc and marg == bm
            allpos = crit + marg + br + be
            assert sorted(allpos) == list(range(n))


# --------------------------------------------------------------------------- attention pins

def _per_head(p, fn):
    H = p.cfg.llm.q_heads
    G = H // p.cfg.llm.kv_heads
    for b in range(p.batch):
        for h in range(H):
            fn(b, h, h // G, int(p.head_map[p.llm_layer_ids[0] * H + h]))


def test_P1_full_budget_is_dense_attention(oracle_mod):
    """K'+R' = n, M = 0 => O = dense attention = torch SDPA."""
    p = _small(seq_lens=(150, 97, 1), budget=(10_000, 17, 0))
    sel, out, wsum = _run(oracle_mod, p)

    def check(b, h, g, j):
        n = int(p.seq_lens[b])
        K = dense_rows(p.llm, 0, b, n, g, "k")
        V = dense_rows(p.llm, 0, b, n, g, "v")
        ref = sdpa_fp64(p.llm_q[0, b, h], K, V)
        np.testing.assert_allclose(out[b, h], ref.numpy(), rtol=1e-12, atol=1e-12)
        assert abs(wsum[b, h] - 1.0) < 1e-12
    _per_head(p, check)


def test_P2_no_marginal_is_topk_eviction(oracle_mod):
    """M = 0 => O = attention over C ∪ R only (plain top-k eviction, BJ;
    S:314) = SDPA with a boolean mask from a brute-force sort."""
    p = _small(seq_lens=(150, 97, 5), budget=(30, 10, 0))
    sel, out, _ = _run(oracle_mod, p)

    def check(b, h, g, j):
        n = int(p.seq_lens[b])
        _, a = _slm_softmax(p, j, b)
        bc, _, br, _ = brute_split(a.tolist(), 30, 10, 0)
        mask = torch.zeros(n, dtype=torch.bool)
        mask[bc + br] = True
        K = dense_rows(p.llm, 0, b, n, g, "k")
        V = dense_rows(p.llm, 0, b, n, g, "v")
        ref = sdpa_fp64(p.llm_q[0, b, h], K, V, mask)
        np.testing.assert_allclose(out[b, h], ref.numpy(), rtol=1e-12, atol=1e-12)
    _per_head(p, check)


def test_P3_marginal_only_is_slm_weights_times_llm_v(oracle_mod):
    """K = R = 0, M = n => O = a'·V_LLM (Eq. 6 second branch everywhere)."""
    p = _small(seq_lens=(150, 97, 1), budget=(0, 0, 10_000))
    sel, out, _ = _run(oracle_mod, p)

    def check(b, h, g, j):
        n = int(p.seq_lens[b])
        _, a = _slm_softmax(p, j, b)
        V = dense_rows(p.llm, 0, b, n, g, "v")
        np.testing.assert_allclose(out[b, h], (a @ V).numpy(), rtol=1e-12, atol=1e-13)
    _per_head(p, check)


def test_empty_selection_gives_zero(oracle_mod):
    """K = R = M = 0: C ∪ R empty => O_c = 0 (R2 reading A11), O_m = 0."""
    p = _small(budget=(0, 0, 0))
    _, out, wsum = _run(oracle_mod, p)
    assert np.all(out == 0.0) and np.all(wsum == 0.0)


def test_P9_additivity(oracle_mod):
    """O(C, M) = O(C, ∅) + Σ_{k∈M} a'_k V_k."""
    p = _small(seq_lens=(150, 97), budget=(30, 10, 40))
    sel, out, _ = _run(oracle_mod, p)
    p0 = dataclasses.replace(p, k_marg=torch.zeros_like(p.k_marg))
    _, out0, _ = _run(oracle_mod, p0)
    rows = list(sel["rows"])

    def check(b, h, g, j):
        r = rows.index(j)
        Mc = int(sel["counts"][r, b, 1])
        M = torch.tensor(sel["marg"][r, b, :Mc].tolist(), dtype=torch.long)
        _, a = _slm_softmax(p, j, b)
        n = int(p.seq_lens[b])
        V = dense_rows(p.llm, 0, b, n, g, "v")
        om = a[M] @ V[M]
        np.testing.assert_allclose(out[b, h] - out0[b, h], om.numpy(), rtol=1e-11, atol=1e-12)
    _per_head(p, check)


def test_P4_slm_equals_llm_closed_form(oracle_mod):
    """SLM ≡ LLM (same q, K, d; identity map): with p the full softmax,
    O - dense = (1/P_{C∪R} - 1) Σ_{C∪R} p V (D2 renormalisation, D3 no
    renormalisation of the spliced row)."""
    cfg = synth.small_config(llm=(1, 4, 2, 64), slm=(1, 4, 2, 64), seq_len=130, batch=2,
                             budget=(20, 8, 30))
    p = synth.make_problem(cfg, seed=3, page_size=16, seq_lens=[130, 61])
    slm = dataclasses.replace(p.slm, k=p.llm.k.clone(), block_table=p.llm.block_table.clone())
    p = dataclasses.replace(p, slm=slm, slm_q=p.llm_q.clone(),
                            head_map=torch.arange(4, dtype=torch.int32))
    sel, out, _ = _run(oracle_mod, p)

    def check(b, h, g, j):
        n = int(p.seq_lens[b])
        K = dense_rows(p.llm, 0, b, n, g, "k")
        V = dense_rows(p.llm, 0, b, n, g, "v")
        s = (K @ p.llm_q[0, b, h].double()) / math.sqrt(64)
        pr = torch.softmax(s, 0)
        dense = pr @ V
        r = list(sel["rows"]).index(j)
        Kc, Mc, Rc = (int(x) for x in sel["counts"][r, b])
        CR = sel["crit"][r, b, :Kc].tolist() + list(range(n - Rc, n))
        P = pr[CR].sum()
        expect = dense + (1.0 / P - 1.0) * (pr[CR] @ V[CR])
        # minus the evicted mass: O = O_CR/P + O_M, dense = O_CR + O_M + O_E
        Mset = sel["marg"][r, b, :Mc].tolist()
        E = sorted(set(range(n)) - set(CR) - set(Mset))
        expect = expect - (pr[E] @ V[E] if E else 0.0)
        np.testing.assert_allclose(out[b, h], expect.numpy(), rtol=1e-11, atol=1e-12)
    _per_head(p, check)


# --------------------------------------------------------------------------- matching (P14)

def test_P14_match_planted_identity(oracle_mod):
    rng = np.random.default_rng(0)
    w, k = 150, 30
    llm_F = rng.random((12, w))
    clone_of = [3, 7, 0, 11]
    slm_F = llm_F[clone_of] * 2.5  # positive rescaling leaves TopK unchanged
    hm, jac = oracle_mod.match_heads(llm_F, slm_F, k)
    for j, i in enumerate(clone_of):
        assert hm[i] == j and jac[i] == 1.0


def test_P14_single_slm_head(oracle_mod):
    rng = np.random.default_rng(1)
    hm, jac = oracle_mod.match_heads(rng.random((9, 120)), rng.random((1, 120)), 24)
    assert np.all(hm == 0)


def test_match_bruteforce_and_ties(oracle_mod):
    """Exhaustive Python-set Jaccard + argmax (smallest j on ties)."""
    rng = np.random.default_rng(2)
    for trial in range(30):
        w = int(rng.integers(8, 40))
        k = int(rng.integers(1, w))
        llm_F = rng.integers(0, 4, (5, w)).astype(float)  # many ties
        slm_F = rng.integers(0, 4, (6, w)).astype(float)
        slm_F[3] = slm_F[1]  # duplicate SLM head: must never win over j=1
        hm, jac = oracle_mod.match_heads(llm_F, slm_F, k)

        def top(F):
            return set(sorted(range(w), key=lambda v: (-F[v], v))[:k])
        for i in range(5):
            sims = [len(top(llm_F[i]) & top(slm_F[j])) / len(top(llm_F[i]) | top(slm_F[j]))
                    for j in range(6)]
            best = max(sims)
            assert hm[i] == sims.index(best) and jac[i] == pytest.approx(best, abs=1e-15)


def test_match_monotone_in_slm_pool(oracle_mod):
    """Adding SLM heads never lowers any best similarity."""
    rng = np.random.default_rng(3)
    llm_F, slm_F = rng.random((10, 100)), rng.random((8, 100))
    _, j4 = oracle_mod.match_heads(llm_F, slm_F[:4], 20)
    _, j8 = oracle_mod.match_heads(llm_F, slm_F, 20)
    assert np.all(j8 >= j4)


# --------------------------------------------------------------------------- f1 (accumulated score)

def test_P13_accumulated_score_uniform_causal(oracle_mod):
    """f1: q' = 0 makes every decode row uniform over its n tokens; three steps
    with n = 1, 2, 3 accumulate the column sums of the uniform causal matrix,
    (11/6, 5/6, 1/3) (Eq. 1)."""
    p = _small(seq_lens=(3,), budget=(1, 0, 1))
    p = dataclasses.replace(p, slm_q=torch.zeros_like(p.slm_q))
    slm, _ = _views(oracle_mod, p)
    rows = oracle_mod.image_rows(p.head_map)
    acc = np.zeros((len(rows), 1, 3), np.float64)
    for n in (1, 2, 3):
        sel = oracle_mod.select_acc(p.slm_q, slm, torch.tensor([n], dtype=torch.int32), rows,
                                    p.k_crit, p.n_recent, p.k_marg, p.max_crit, p.max_marg, 3,
                                    acc)
    g = GOLDEN["column_sums_uniform_causal_n3"]["F"]
    np.testing.assert_allclose(acc[:, 0, :], np.tile(g, (len(rows), 1)), rtol=0, atol=1e-15)
    # ranked by the running sums: position 0 (11/6) is critical, 1 (5/6) marginal
    assert sel["crit"][0, 0, 0] == 0 and sel["marg"][0, 0, 0] == 1


def test_f1_accumulated_equals_sum_of_rows(oracle_mod):
    """acc after T steps = Σ_t softmax rows (torch), and the sets = full sort of it."""
    p = _small(seq_lens=(90, 60), budget=(10, 5, 15))
    slm, _ = _views(oracle_mod, p)
    rows = oracle_mod.image_rows(p.head_map)
    acc = np.zeros((len(rows), 2, 90), np.float64)
    ref = np.zeros_like(acc)
    steps = [(80, 50), (85, 55), (90, 60)]
    for ns in steps:
        sl = torch.tensor(ns, dtype=torch.int32)
        sel = oracle_mod.select_acc(p.slm_q, slm, sl, rows, p.k_crit, p.n_recent, p.k_marg,
                                    p.max_crit, p.max_marg, 90, acc)
        pp = dataclasses.replace(p, seq_lens=sl)
        for r, j in enumerate(rows):
            for b in range(2):
                _, a = _slm_softmax(pp, j, b)
                ref[r, b, :ns[b]] += a.numpy()
    np.testing.assert_allclose(acc, ref, rtol=1e-12, atol=1e-15)
    for r in range(len(rows)):
        for b in range(2):
            n = steps[-1][b]
            bc, bm, _, _ = brute_split(ref[r, b, :n].tolist(), 10, 5, 15)
            Kc, Mc, _ = sel["counts"][r, b]
            assert sel["crit"][r, b, :Kc].tolist() == bc
            assert sel["marg"][r, b, :Mc].tolist() == bm


# --------------------------------------------------------------------------- variant f2
def _group_map(p, kind):
    """Head map for f2 pins: "uniform" = every head of an LLM kv group maps to
    one SLM row; else the problem's own (random) map."""
    if kind != "uniform":
        return p
    H, H_kv = p.cfg.llm.q_heads, p.cfg.llm.kv_heads
    G = H // H_kv
    n_slm = p.cfg.slm.layers * p.cfg.slm.q_heads
    rng = random.Random(7)
    hm = torch.empty(p.cfg.llm.layers * H, dtype=torch.int32)
    for lg in range(p.cfg.llm.layers * H_kv):
        hm[lg * G:(lg + 1) * G] = rng.randrange(n_slm)
    return dataclasses.replace(p, head_map=hm)


def _run_group(oracle, p, layer_slot=0):
    slm, llm = _views(oracle, p)
    rows = oracle.image_rows(p.head_map)
    n_slm = p.cfg.slm.layers * p.cfg.slm.q_heads
    sel = oracle.select(p.slm_q, slm, p.seq_lens, rows, p.k_crit, p.n_recent, p.k_marg,
                        p.max_crit, p.max_marg, p.max_seq_len)
    layer = p.llm_layer_ids[layer_slot]
    gsel = oracle.select_group(layer, p.cfg.llm.q_heads, p.cfg.llm.kv_heads, p.head_map, sel,
                               p.seq_lens, p.k_crit, p.n_recent, p.k_marg, p.max_crit,
                               p.max_marg, n_slm)
    out, wsum = oracle.attend_group(layer, layer_slot, p.llm_q[layer_slot], llm, p.seq_lens,
                                    p.head_map, sel, gsel, n_slm)
    return sel, gsel, out, wsum


def test_P16_f2_uniform_group_reduces_to_default(oracle_mod):
    """f2 with every head of a group on one SLM row: F_g = G·a' (an exact
    power-of-two scale for G=4) ranks like a' => the default method."""
    p = _group_map(_small(seq_lens=(150, 97, 1), budget=(30, 10, 40)), "uniform")
    sel, gsel, out_g, wsum_g = _run_group(oracle_mod, p)
    _, out, wsum = _run(oracle_mod, p)
    np.testing.assert_array_equal(out_g, out)
    np.testing.assert_array_equal(wsum_g, wsum)


def test_P17_f2_group_split_bruteforce(oracle_mod):
    """f2 split = Python sort of the torch-softmax rows summed over the group's
    heads (R16: F_g = Σ_h a'_{f(h)})."""
    p = _small(seq_lens=(150, 97, 5), budget=(30, 10, 40))
    _, gsel, _, _ = _run_group(oracle_mod, p)
    H, H_kv = p.cfg.llm.q_heads, p.cfg.llm.kv_heads
    G = H // H_kv
    layer = p.llm_layer_ids[0]
    for g in range(H_kv):
        for b in range(p.batch):
            F = sum(_slm_softmax(p, int(p.head_map[layer * H + g * G + h]), b)[1] for h in range(G))
            bc, bm, br, _ = brute_split(F.tolist(), 30, 10, 40)
            Kc, Mc, Rc = (int(x) for x in gsel["counts"][g, b])
            assert (Kc, Mc, Rc) == (len(bc), len(bm), len(br))
            assert gsel["crit"][g, b, :Kc].tolist() == bc
            assert gsel["marg"][g, b, :Mc].tolist() == bm


def test_P18_f2_attend_shared_sets_own_weights(oracle_mod):
    """f2 attention: M = 0 => SDPA over the group's shared C ∪ R (mask from the
    brute-force split of F_g); K = R = 0 => Σ_{k∈M_g} a'_{f(h)}[k] V[k] with the
    head's OWN row weights (Eq. 6 second branch)."""
    H, H_kv = 8, 2
    G = H // H_kv
    for budget in ((30, 10, 0), (0, 0, 60)):
        p = _small(seq_lens=(150, 97, 5), budget=budget)
        _, _, out, _ = _run_group(oracle_mod, p)
        layer = p.llm_layer_ids[0]
        for b in range(p.batch):
            n = int(p.seq_lens[b])
            for g in range(H_kv):
                F = sum(_slm_softmax(p, int(p.head_map[layer * H + g * G + h]), b)[1]
                        for h in range(G))
                bc, bm, br, _ = brute_split(F.tolist(), *budget)
                K = dense_rows(p.llm, 0, b, n, g, "k")
                V = dense_rows(p.llm, 0, b, n, g, "v")
                for h in range(g * G, (g + 1) * G):
                    if budget[2] == 0:
                        mask = torch.zeros(n, dtype=torch.bool)
                        mask[bc + br] = True
                        ref = sdpa_fp64(p.llm_q[0, b, h], K, V, mask)
                    else:
                        _, a = _slm_softmax(p, int(p.head_map[layer * H + h]), b)
                        w = torch.zeros(n, dtype=torch.float64)
                        w[bm] = a[bm]
                        ref = w @ V
                    np.testing.assert_allclose(out[b, h], ref.numpy(), rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- variant f3
def test_P19_f3_matching_window_spec(oracle_mod):
    """R17 window: SPEC's worked decisions: 50 -> DEFER, 150 ->
    [0,150), 1000 -> [800,1000) (keep the most recent); first-w reading -> [0,200)."""
    w = GOLDEN["matching_window"]
    for n, want in w["cases"]:
        got = oracle_mod.match_window(n, w["min_len"], w["max_len"], keep_last=True)
        assert (None if got is None else [got[0], got[0] + got[1]]) == want
    assert oracle_mod.match_window(1000, 100, 200, keep_last=False) == (0, 200)
    assert oracle_mod.match_window(100, 100, 200) == (0, 100)
    assert oracle_mod.match_window(99, 100, 200) is None


def _prefill_problem(n, seed=3):
    cfg = synth.small_config(llm=(2, 8, 2, 64), slm=(2, 4, 2, 64), seq_len=n, batch=2,
                             budget=(10, 5, 10))
    return synth.make_problem(cfg, seed=seed, page_size=16, seq_lens=[n, n])


def test_P20_f3_uniform_causal_column_sums(oracle_mod):
    """q = 0 => every causal row is uniform over its prefix => F = column sums
    of the uniform causal matrix: (11/6, 5/6, 1/3) for the first 3 tokens
    (S:61), and Σ_{u>=v} 1/(start+u+1) for a window starting later."""
    p = _prefill_problem(40)
    _, llm = _views(oracle_mod, p)
    H, d = p.cfg.llm.q_heads, p.cfg.llm.head_dim
    for start, length in ((0, 3), (25, 15)):
        q = torch.zeros(p.llm.num_layers, length, H, d, dtype=torch.bfloat16)
        F = oracle_mod.prefill_scores(q, llm, 1, start, length)
        ref = np.array([sum(1.0 / (start + u + 1) for u in range(v, length)) for v in range(length)])
        np.testing.assert_allclose(F, np.broadcast_to(ref, F.shape), rtol=1e-13, atol=0)
        if start == 0:
            np.testing.assert_allclose(F[0], GOLDEN["column_sums_uniform_causal_n3"]["F"],
                                       rtol=1e-13)


def test_P21_f3_prefill_scores_vs_torch(oracle_mod):
    """F = torch softmax of the causally masked q·K^T/sqrt(d) over the full
    prefix, summed over the window's rows, window columns (Eq. 1)."""
    p = _prefill_problem(60)
    _, llm = _views(oracle_mod, p)
    H, d, G = p.cfg.llm.q_heads, p.cfg.llm.head_dim, p.cfg.llm.q_heads // p.cfg.llm.kv_heads
    g = torch.Generator().manual_seed(5)
    for start, length in ((0, 60), (37, 23)):
        q = torch.randn(p.llm.num_layers, length, H, d, generator=g).to(torch.bfloat16)
        F = oracle_mod.prefill_scores(q, llm, 0, start, length)
        for l in range(p.llm.num_layers):
            for h in range(H):
                K = dense_rows(p.llm, l, 0, start + length, h // G, "k")
                s = (q[l, :, h].double() @ K.T) / math.sqrt(d)
                pos = torch.arange(start, start + length).view(-1, 1)
                s = s.masked_fill(torch.arange(start + length).view(1, -1) > pos, float("-inf"))
                ref = torch.softmax(s, dim=1).sum(0)[start:]
                np.testing.assert_allclose(F[l * H + h], ref.numpy(), rtol=1e-12, atol=1e-14)
