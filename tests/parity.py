"""Parity machinery shared by the GPU tests, smoke() and bench.py's checks.

Compares the CUDA path (through the C ABI) with the fp64 oracle on the same
seeded inputs, per the bars of DESIGN.md §5:
  * index sets bit-exact except tokens whose oracle score lies within
    1e-6·max(1,|θ|) of a rank boundary θ (A18); counts exactly equal;
  * outputs row-normwise max relative error <= 2e-3 (A19), with the oracle
    evaluated on the GPU's verified sets.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

SET_BAND = 1e-6          # BASELINE.json north_star: score gaps below 1e-6 are exempt
FLIP_LOGIT_BAND = 2e-5   # stricter internal bar: flips only within fp32 logit rounding
OUT_TOL = 2e-3


def views(p):
    slm = oracle.CacheView(p.slm.k, None, p.slm.block_table, p.slm.num_pages, p.slm.page_size,
                           p.slm.num_layers, p.cfg.slm.q_heads, p.cfg.slm.kv_heads,
                           p.cfg.slm.head_dim)
    llm = oracle.CacheView(p.llm.k, p.llm.v, p.llm.block_table, p.llm.num_pages,
                           p.llm.page_size, p.llm.num_layers, p.cfg.llm.q_heads,
                           p.cfg.llm.kv_heads, p.cfg.llm.head_dim)
    return slm, llm


def oracle_select(p, rows=None, slm_view=None):
    slm = slm_view or views(p)[0]
    rows = oracle.image_rows(p.head_map) if rows is None else np.asarray(rows, np.int32)
    return oracle.select(p.slm_q, slm, p.seq_lens, rows, p.k_crit, p.n_recent, p.k_marg,
                         p.max_crit, p.max_marg, p.max_seq_len)


def compare_select(p, gpu, sel, rows=None, batch_idx=None, logit_atol=2e-4, rank_score=None):
    """Check GPU select outputs against oracle dict `sel` for its rows.
    rank_score: the oracle's ranking score per [row][b][v] when it is not the
    current-row probability (variant f1: the running sums); flips are then
    bounded relative to it.  Returns a report dict; raises AssertionError."""
    rows = sel["rows"]
    lg = gpu.logits.cpu().double().numpy()
    lse = gpu.lse.cpu().double().numpy()
    crit = gpu.crit.cpu().numpy()
    marg = gpu.marg.cpu().numpy()
    mw = gpu.marg_w.cpu().double().numpy()
    cnt = gpu.counts.cpu().numpy()
    bs = range(p.batch) if batch_idx is None else batch_idx
    rep = {"max_logit_err": 0.0, "max_lse_err": 0.0, "exempt_tokens": 0, "rows_checked": 0,
           "max_margw_rel": 0.0, "flips": 0, "max_flip_logit_gap": 0.0}
    for r, j in enumerate(rows):
        for b in bs:
            n = int(p.seq_lens[b])
            o_s = sel["s"][r, b, :n]
            o_a = sel["a"][r, b, :n]
            o_r = o_a if rank_score is None else rank_score[r, b, :n]   # ranking score
            Kc, Mc, Rc = (int(x) for x in sel["counts"][r, b])
            err = np.abs(lg[j, b, :n] - o_s).max()
            rep["max_logit_err"] = max(rep["max_logit_err"], float(err))
            assert err <= logit_atol, f"logits row {j} seq {b}: {err}"
            m, l_ = sel["stats"][r, b]
            e2 = max(abs(lse[j, b, 0] - m), abs(lse[j, b, 1] - l_))
            rep["max_lse_err"] = max(rep["max_lse_err"], float(e2))
            assert e2 <= 1e-4, f"lse row {j} seq {b}: {e2}"
            assert cnt[j, b, 0] == Kc and cnt[j, b, 1] == Mc, (j, b, cnt[j, b], Kc, Mc)
            gC = crit[j, b, :Kc]
            gM = marg[j, b, :Mc]
            assert np.all(np.diff(gC) > 0) and np.all(np.diff(gM) > 0), "lists not ascending"
            oC = set(sel["crit"][r, b, :Kc].tolist())
            oM = set(sel["marg"][r, b, :Mc].tolist())
            # exempt band around the oracle's two rank boundaries
            ranked = np.sort(o_r[: n - Rc])[::-1]
            exempt = np.zeros(n, bool)
            for k in (Kc, Kc + Mc):
                if 0 < k <= n - Rc:
                    th = ranked[k - 1]
                    exempt |= np.abs(o_r - th) < SET_BAND * max(1.0, abs(th))
            exempt[n - Rc:] = False
            ex = set(np.nonzero(exempt)[0].tolist())
            rep["exempt_tokens"] += len(ex)
            assert set(gC.tolist()) - ex == oC - ex, f"critical set mismatch row {j} seq {b}"
            assert set(gM.tolist()) - ex == oM - ex, f"marginal set mismatch row {j} seq {b}"
            # stricter than the bar: tokens actually classified differently must
            # sit within fp32 logit rounding (FLIP_LOGIT_BAND) of a boundary logit
            flipped = (set(gC.tolist()) ^ oC) | (set(gM.tolist()) ^ oM)
            if flipped:
                sc = o_s if rank_score is None else o_r   # logits, or the f1 sums
                bounds = [sc[np.argsort(-o_r[: n - Rc], kind="stable")[k - 1]]
                          for k in (Kc, Kc + Mc) if 0 < k <= n - Rc]
                gap = max(min(abs(sc[v] - t) / max(1.0, abs(t)) for t in bounds)
                          for v in flipped)
                rep["flips"] += len(flipped)
                rep["max_flip_logit_gap"] = max(rep["max_flip_logit_gap"], float(gap))
                assert gap <= FLIP_LOGIT_BAND, f"flip {gap} away from a boundary, row {j} seq {b}"
            assert not (set(gC.tolist()) & set(gM.tolist()))
            assert np.all(gC < n - Rc) and np.all(gM < n - Rc)
            if Mc:
                ref = o_a[gM]
                # fp32 output (R15): weights below fp32's normal range (1e-38) cannot
                # be represented, so they are compared absolutely at 1e-30 scale
                rel = np.abs(mw[j, b, :Mc] - ref) / np.maximum(ref, 1e-30)
                rep["max_margw_rel"] = max(rep["max_margw_rel"], float(rel.max()))
                assert rel.max() <= 1e-4, f"marg_w row {j} seq {b}: {rel.max()}"
            rep["rows_checked"] += 1
    return rep


def sel_from_gpu(p, gpu, sel):
    """The oracle's selection dict with the GPU's (verified) lists substituted,
    so the output check does not depend on permitted boundary flips (A19)."""
    rows = sel["rows"]
    crit = gpu.crit.cpu().numpy()[rows]
    marg = gpu.marg.cpu().numpy()[rows]
    counts = sel["counts"].copy()
    return {"rows": rows, "a": sel["a"], "crit": crit, "marg": marg, "counts": counts}


def row_normwise(o, ref):
    num = np.abs(o - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-30)
    return num / den


def compare_attend(p, layer_slot, out_gpu, sel_gpu_sets, llm_view=None, heads=None):
    llm = llm_view or views(p)[1]
    layer = p.llm_layer_ids[layer_slot]
    ref, wsum = oracle.attend(layer, layer_slot, p.llm_q[layer_slot], llm, p.seq_lens,
                              p.head_map, sel_gpu_sets, p.cfg.slm.layers * p.cfg.slm.q_heads)
    o = out_gpu.cpu().double().numpy()
    err = row_normwise(o, ref)
    if heads is not None:
        err = err[heads]
    return float(err.max()), ref


def run_gpu_step(p, step=None, layers=None):
    """select + attend for the resident layers; returns (step, select_out, outs)."""
    from paper_2508_02751_b200 import smallkv
    step = step or smallkv.from_problem(p)
    sel = step.select(p.slm_q)
    outs = []
    for i, slot in enumerate(range(p.llm.num_layers) if layers is None else layers):
        out = torch.empty(p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim, dtype=torch.float32,
                          device=p.seq_lens.device)
        # later layers may overlap their prologue with the previous attend (PDL)
        step.attend(p.llm_layer_ids[slot], slot, p.llm_q[slot], out, overlap_prologue=i > 0)
        outs.append(out)
    torch.cuda.synchronize()
    return step, sel, outs


# --------------------------------------------------------------------------- variant f2
def compare_group(p, gpu, sel, layer_slot, out_gpu=None, llm_view=None):
    """Variant f2 (R16): the GPU's group selection of LLM layer
    p.llm_layer_ids[layer_slot] (smallkv_select_group outputs `gpu`) against
    oracle_select_group, the per-head marginal weights against the oracle's
    rows a'_{f(h)}, and (if out_gpu is given) the attention output against
    oracle_attend_group evaluated on the GPU's verified sets."""
    H, H_kv = p.cfg.llm.q_heads, p.cfg.llm.kv_heads
    G = H // H_kv
    n_slm = p.cfg.slm.layers * p.cfg.slm.q_heads
    layer = p.llm_layer_ids[layer_slot]
    gsel = oracle.select_group(layer, H, H_kv, p.head_map, sel, p.seq_lens, p.k_crit, p.n_recent,
                               p.k_marg, p.max_crit, p.max_marg, n_slm)
    slot_of = {int(j): r for r, j in enumerate(sel["rows"])}
    hm = p.head_map.cpu().numpy()
    score = gpu.logits.cpu().double().numpy()
    crit = gpu.crit.cpu().numpy()
    marg = gpu.marg.cpu().numpy()
    mw8 = gpu.marg_w.cpu().double().numpy()
    cnt = gpu.counts.cpu().numpy()
    rep = {"max_score_err": 0.0, "flips": 0, "exempt_tokens": 0, "max_margw_rel": 0.0,
           "groups_checked": 0}
    g_crit = np.zeros_like(gsel["crit"])
    g_marg = np.zeros_like(gsel["marg"])
    for g in range(H_kv):
        gl = layer * H_kv + g
        for b in range(p.batch):
            n = int(p.seq_lens[b])
            F = gsel["score"][g, b, :n]
            Kc, Mc, Rc = (int(x) for x in gsel["counts"][g, b])
            err = np.abs(score[gl, b, :n] - F).max() if n else 0.0
            rep["max_score_err"] = max(rep["max_score_err"], float(err))
            assert err <= 1e-5 * max(1.0, float(F.max())), f"group score {gl} seq {b}: {err}"
            assert cnt[gl, b, 0] == Kc and cnt[gl, b, 1] == Mc, (gl, b, cnt[gl, b], Kc, Mc)
            gC, gM = crit[gl, b, :Kc], marg[gl, b, :Mc]
            assert np.all(np.diff(gC) > 0) and np.all(np.diff(gM) > 0), "lists not ascending"
            oC = set(gsel["crit"][g, b, :Kc].tolist())
            oM = set(gsel["marg"][g, b, :Mc].tolist())
            order = np.argsort(-F[: n - Rc], kind="stable")
            bounds = [F[order[k - 1]] for k in (Kc, Kc + Mc) if 0 < k <= n - Rc]
            exempt = np.zeros(n, bool)
            for th in bounds:
                exempt |= np.abs(F - th) < SET_BAND * max(1.0, abs(th))
            exempt[n - Rc:] = False
            ex = set(np.nonzero(exempt)[0].tolist())
            rep["exempt_tokens"] += len(ex)
            assert set(gC.tolist()) - ex == oC - ex, f"f2 critical set mismatch {gl} seq {b}"
            assert set(gM.tolist()) - ex == oM - ex, f"f2 marginal set mismatch {gl} seq {b}"
            flipped = (set(gC.tolist()) ^ oC) | (set(gM.tolist()) ^ oM)
            if flipped:
                gap = max(min(abs(F[v] - t) / max(1.0, abs(t)) for t in bounds) for v in flipped)
                rep["flips"] += len(flipped)
                assert gap <= FLIP_LOGIT_BAND, f"f2 flip {gap} away from a boundary {gl} seq {b}"
            assert not (set(gC.tolist()) & set(gM.tolist()))
            for m in range(Mc):
                for h in range(8):
                    w = mw8[gl, b, m, h]
                    if h >= G:
                        assert w == 0.0
                        continue
                    j = int(hm[layer * H + g * G + h])
                    ref = sel["a"][slot_of[j], b, gM[m]]
                    rel = abs(w - ref) / max(ref, 1e-300)
                    rep["max_margw_rel"] = max(rep["max_margw_rel"], float(rel))
                    assert rel <= 1e-4, f"f2 marg_w {gl} seq {b} m {m} h {h}: {rel}"
            g_crit[g, b, :Kc] = gC
            g_marg[g, b, :Mc] = gM
            rep["groups_checked"] += 1
    if out_gpu is not None:
        llm = llm_view or views(p)[1]
        gsets = {"crit": g_crit, "marg": g_marg, "counts": gsel["counts"]}
        ref, _ = oracle.attend_group(layer, layer_slot, p.llm_q[layer_slot], llm, p.seq_lens,
                                     p.head_map, sel, gsets, n_slm)
        err = row_normwise(out_gpu.cpu().double().numpy(), ref)
        rep["max_out_err"] = float(err.max())
        assert err.max() <= OUT_TOL, f"f2 output error {err.max()}"
    return rep


def attend_split(step) -> int:
    """CTAs per (sequence, kv-group) the attend of a DecodeStep launches (under
    the stream-K split: the record slots, the most shares a group has),
    recovered from smallkv_plan_size: L*B*H_kv records of 256 + NC * (384 +
    1024 x 12) bytes (gather_attend.cu plan_record_bytes)."""
    import ctypes
    L = step.llm_layers
    nb = step.lib.smallkv_plan_size(ctypes.byref(step.llm), ctypes.byref(step.batch), L)
    per = nb // (L * step.batch.batch * step.llm.num_kv_heads)
    return (per - 256) // (384 + 1024 * 12)


def assert_same_outputs(a, b, same_split: bool):
    """Bitwise when both runs split the groups' lists alike; otherwise equal up
    to the fp32 rounding of the split-merge order, row-normwise <= 1e-5
    (DESIGN.md §5)."""
    if same_split:
        assert torch.equal(a, b)
    else:
        err = row_normwise(a.double().cpu().numpy(), b.double().cpu().numpy()).max()
        assert err <= 1e-5, err
