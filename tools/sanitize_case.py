"""Small decode steps through every launch chain, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_case.py

Runs (through the C ABI, on tiny shapes so the instrumented kernels finish in
seconds): the toy config (BASELINE configs[0]); a small ragged config over the
default chain row_flags -> K1 -> K2 -> plan -> attend x L with the PDL overlap
prologue; the same without a plan; K1/K2 in SLM-layer chunks with K2 on an
auxiliary stream; variant f1 (accumulated scores); f2 (group selection);
f4 (tiered pool, including a capacity overflow); f3 prefill scores + K0.
Outputs are not checked here (the parity tests do that); the sanitizer's
report is the result.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import smallkv_synth as synth  # noqa: E402
from paper_2508_02751_b200 import smallkv  # noqa: E402


def step_all(p, **kw):
    st = smallkv.from_problem(p, **kw)
    st.select(p.slm_q)
    for i, slot in enumerate(range(p.llm.num_layers)):
        out = torch.empty(p.batch, p.cfg.llm.q_heads, p.cfg.llm.head_dim, device="cuda")
        st.attend(p.llm_layer_ids[slot], slot, p.llm_q[slot], out, overlap_prologue=i > 0)
    torch.cuda.synchronize()
    return st


def main():
    torch.cuda.set_device(0)
    which = sys.argv[1:] or ["toy", "default", "noplan", "aux", "f1", "f2", "f4", "f3"]
    toy = synth.make_problem(synth.CONFIGS["toy"], seed=0).to("cuda")
    cfg = synth.small_config(llm=(2, 8, 2, 128), slm=(3, 8, 2, 64), seq_len=2100, batch=3,
                             budget=(150, 60, 200))
    p = synth.make_problem(cfg, seed=5, page_size=16, seq_lens=[2100, 700, 1],
                           map_kind="random").to("cuda")
    # a long row (> 8192 tokens: the global-memory select variant) in one sequence
    cfg_l = synth.small_config(llm=(1, 8, 2, 128), slm=(1, 4, 1, 64), seq_len=9000, batch=1,
                               budget=(900, 450, 900))
    pl = synth.make_problem(cfg_l, seed=6, page_size=64).to("cuda")
    if "toy" in which:
        step_all(toy)
        print("toy ok", flush=True)
    if "default" in which:
        step_all(p)
        step_all(pl)
        print("default ok", flush=True)
    if "noplan" in which:
        step_all(p, use_plan=False)
        print("noplan ok", flush=True)
    if "aux" in which:
        step_all(p, overlap_select=True)
        print("aux ok", flush=True)
    if "f1" in which:
        st = smallkv.from_problem(p)
        acc = torch.zeros_like(st.out.logits)
        for _ in range(2):
            st.select(p.slm_q, acc=acc)
        torch.cuda.synchronize()
        print("f1 ok", flush=True)
    if "f2" in which:
        step_all(p, variant="f2")
        print("f2 ok", flush=True)
    if "f4" in which:
        for cap_scale in (1, 0):   # 0: capacity below the list size (overflow path)
            st = smallkv.from_problem(p, use_plan=False)
            hk = torch.empty(p.llm.k.shape, dtype=p.llm.k.dtype, pin_memory=True)
            hv = torch.empty(p.llm.v.shape, dtype=p.llm.v.dtype, pin_memory=True)
            hk.copy_(p.llm.k)
            hv.copy_(p.llm.v)
            G = cfg.llm.q_heads // cfg.llm.kv_heads
            cap = -(-(int(p.n_recent.max()) + G * (p.max_crit + p.max_marg)) // 4) * 4
            if cap_scale == 0:
                cap = 64
            tier = smallkv.TieredKV(st, hk, hv, capacity=cap)
            st.select(p.slm_q)
            tier.update()
            for slot in range(p.llm.num_layers):
                out = torch.empty(p.batch, cfg.llm.q_heads, cfg.llm.head_dim, device="cuda")
                tier.attend(slot, p.llm_q[slot], out, overlap_prologue=slot > 0)
            torch.cuda.synchronize()
            if cap_scale == 0:
                assert tier.counters()[1] > 0
                # the first two sequences' lists exceed 64 slots (NaN heads); the
                # one-token sequence fits (finite)
                assert torch.isnan(out[:2]).all(), "overflowed groups must read as NaN"
                assert torch.isfinite(out[2]).all(), "a group that fits must be finite"
        print("f4 ok", flush=True)
    if "f3" in which:
        g = torch.Generator(device="cuda").manual_seed(1)
        q = torch.randn(p.slm.num_layers, 150, cfg.slm.q_heads, cfg.slm.head_dim, device="cuda",
                        generator=g).to(torch.bfloat16)
        F = smallkv.prefill_scores(q, p.slm.k, p.slm.block_table, cfg.slm.q_heads, 0, 10)
        ql = torch.randn(p.llm.num_layers, 150, cfg.llm.q_heads, cfg.llm.head_dim, device="cuda",
                         generator=g).to(torch.bfloat16)
        Fl = smallkv.prefill_scores(ql, p.llm.k, p.llm.block_table, cfg.llm.q_heads, 0, 10)
        smallkv.match_heads(Fl, F, 30)
        torch.cuda.synchronize()
        print("f3 ok", flush=True)
    print("sanitize_case done", flush=True)


if __name__ == "__main__":
    main()
