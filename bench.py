#!/usr/bin/env python
"""Benchmark of the SmallKV decode hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config qwen7b]

A step = one pass of the whole hot path over one batch: smallkv_select over
all SLM layers (K1 score + K2 split) and one smallkv_attend per LLM layer
(K3 gather-attend with the fused combine), captured in one CUDA graph.
Metric (BASELINE.json): decode-attention layer-steps/s (= L LLM layers per
step) and achieved HBM GB/s over the algorithmic bytes of DESIGN.md §7.
Default workload: BASELINE.json configs[1] (Qwen2.5-7B + Qwen2.5-0.5B, ctx 4096,
batch 32 per GPU).  N > 1 (torchrun, one rank per GPU): batch sharding, every
rank runs its own batch (weak scaling), no data-path collective; the step time
is the max over ranks (device clock, CUDA events).

`--impl reference` times the fp64 CPU oracle (oracle/) as the reference arm on
a bounded sample of the same workload; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "decode attn layer-steps/s and achieved HBM GB/s vs ~8 TB/s, at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(gpu_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(cfg_name: str, rank: int, world: int, shard: str, device):
    """This rank's inputs.  batch sharding: its own batch of cfg.batch sequences
    (seed = rank, weak scaling).  head sharding: the shared batch (seed 0) with
    the LLM side restricted to this rank's kv-groups (strong scaling)."""
    import dataclasses
    import torch
    import smallkv_synth as synth
    from paper_2508_02751_b200 import dist as pdist
    cfg = synth.CONFIGS[cfg_name]
    heads = shard in ("heads", "heads-slm") and world > 1
    kv_share = cfg.llm.kv_heads // world if heads else cfg.llm.kv_heads
    # resident LLM layers: all when they fit, else a rotating subset (each slice >> L2)
    per_layer = cfg.batch * kv_share * cfg.seq_len * cfg.llm.head_dim * 2 * 2
    free = torch.cuda.mem_get_info(device)[0]
    slm_bytes = cfg.slm.layers * cfg.batch * cfg.slm.kv_heads * cfg.seq_len * cfg.slm.head_dim * 2
    budget = int(0.8 * free) - slm_bytes - (4 << 30)
    if heads:   # the full LLM pool is generated once, then sliced
        budget = budget * kv_share // cfg.llm.kv_heads
    resident = max(1, min(cfg.llm.layers, budget // per_layer))
    p = synth.make_problem(cfg, seed=0 if heads else rank, device=device,
                           llm_layers=list(range(resident)))
    if heads:
        g0, g1 = pdist.kv_group_range(cfg.llm.kv_heads, world, rank)
        L, H, Hkv = cfg.llm.layers, cfg.llm.q_heads, cfg.llm.kv_heads
        k, v, q, hm = pdist.slice_llm_kv_groups(p.llm.k, p.llm.v, p.llm_q, p.head_map, L, H,
                                                Hkv, g0, g1)
        dims = synth.ModelDims(L, (g1 - g0) * (H // Hkv), g1 - g0, cfg.llm.head_dim)
        full_hm = p.head_map
        p = dataclasses.replace(p, cfg=dataclasses.replace(cfg, llm=dims),
                                llm=dataclasses.replace(p.llm, k=k, v=v, dims=dims),
                                llm_q=q, head_map=hm)
        p.full_head_map = full_hm   # f3b: the SLM row blocks are cut from the full map
        torch.cuda.empty_cache()
    return p, resident


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    from paper_2508_02751_b200 import build as kbuild
    if rank == 0:
        kbuild.build()
    if world > 1:
        dist.barrier()
    from paper_2508_02751_b200 import bytes_model, smallkv

    heads = args.shard in ("heads", "heads-slm") and world > 1
    slm_part = args.shard == "heads-slm" and world > 1
    p, resident = build_problem(args.config, rank, world, args.shard, device)
    cfg = p.cfg
    L = cfg.llm.layers
    tier = None
    if args.variant == "f4":
        # host-tiered pool: the LLM K/V in pinned host memory,
        # each group's needed rows in an HBM hot pool refreshed per layer
        assert resident == L, "f4 keeps one hot-pool slot per LLM layer"
        step = smallkv.from_problem(p, use_plan=False)
        host_k = torch.empty(p.llm.k.shape, dtype=p.llm.k.dtype, pin_memory=True)
        host_v = torch.empty(p.llm.v.shape, dtype=p.llm.v.dtype, pin_memory=True)
        host_k.copy_(p.llm.k)
        host_v.copy_(p.llm.v)
        # slots per group = the largest list: R' + (#distinct SLM rows of the group) * (K'+M')
        H, Hkv = cfg.llm.q_heads, cfg.llm.kv_heads
        hm = p.head_map.cpu().view(L, Hkv, H // Hkv)
        rows_max = max(len(set(hm[l, g].tolist())) for l in range(L) for g in range(Hkv))
        cap = -(-(int(p.n_recent.max()) + rows_max * (p.max_crit + p.max_marg)) // 4) * 4
        tier = smallkv.TieredKV(step, host_k, host_v, capacity=cap)
    else:
        step = smallkv.from_problem(p, variant=args.variant)
    outs = torch.empty(L, p.batch, cfg.llm.q_heads, cfg.llm.head_dim, dtype=torch.float32,
                       device=device)
    plan = [(l, l % resident, p.llm_q[l % resident], outs[l]) for l in range(L)]
    graph = smallkv.DecodeGraph(step, p.slm_q, plan, timing=False, tier=tier)
    if slm_part:
        # f3b: this rank scores / splits only its block of SLM rows, the blocks
        # are all-gathered (NCCL), then the plan and this rank's kv-group attends
        # run on the exchanged selection; the step runs eagerly (collective inside)
        from paper_2508_02751_b200 import dist as pdist
        n_slm = cfg.slm.layers * cfg.slm.q_heads
        j0, j1 = pdist.slm_row_block(n_slm, world, rank)
        shm = pdist.select_head_map(p.full_head_map.to(device), j0, j1)

        def replay_f3b():
            with torch.cuda.stream(graph.stream):
                step.select(p.slm_q, select_head_map=shm, plan=False)
                pdist.exchange_selection(step.out, n_slm)
                step.plan()
                for i, (layer, slot, q, out) in enumerate(plan):
                    step.attend(layer, slot, q, out, overlap_prologue=i > 0)
        graph.replay = replay_f3b
    if heads:
        # the exchange step of head sharding: all-gather every layer's per-head
        # outputs [L, B, H/w, d] -> [L, B, H, d] once per step (NCCL / NVLink)
        from paper_2508_02751_b200 import dist as pdist
        inner = graph.replay

        def replay_and_gather():
            inner()
            with torch.cuda.stream(graph.stream):
                pdist.gather_heads(outs)
        graph.replay = replay_and_gather
    if args.quick:
        for _ in range(args.warmup):
            graph.replay()
        graph.stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(graph.stream)
        for _ in range(args.steps):
            graph.replay()
        e1.record(graph.stream)
        e1.synchronize()
        if rank == 0:
            print(json.dumps({"quick": True, "ms_per_step": e0.elapsed_time(e1) / args.steps,
                              "kernels_per_step": graph.kernels_per_step}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    sgraph = smallkv.DecodeGraph(step, p.slm_q, [], timing=False)   # select only

    seq = [int(x) for x in p.seq_lens.cpu()]
    buds = list(zip(p.k_crit.cpu().tolist(), p.n_recent.cpu().tolist(), p.k_marg.cpu().tolist()))
    bm = bytes_model.step_bytes_coherent(cfg, seq, buds, L)
    s = graph.stream

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up
    for _ in range(args.warmup):
        graph.replay()
    s.synchronize()
    barrier()

    # ---- timed region: K back-to-back graph replays (device clock); the clock
    # sampler runs from ~0.5 s before it to >= 1.5 s after its start, under the
    # same load
    sampler = ClockSampler(local)
    t_clock0 = time.time()
    while time.time() - t_clock0 < 0.5:
        for _ in range(20):
            graph.replay()
        s.synchronize()
    torch.cuda.synchronize()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    for _ in range(args.steps):
        graph.replay()
    ev1.record(s)
    ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    # keep the clock sampler under the same load for >= 1 s if the region was short
    while time.time() - t_clock0 < 1.5:
        for _ in range(20):
            graph.replay()
        s.synchronize()
    clocks = sampler.stop()

    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    units = 1 if heads else world       # batches processed per step by the whole job
    layer_steps = units * L * args.steps / (max_ms / 1e3)

    # ---- per-kernel durations.  The attend launches of a step overlap through
    # programmatic dependent launch, so an attend's effective duration is
    # measured as (step - select) / L, with select timed alone (same stream,
    # CUDA events, back-to-back replays); the isolated per-launch durations
    # are in the ncu launch list under profiles/.
    nsel = max(20, min(args.steps, 200))
    for _ in range(3):
        sgraph.replay()
    sgraph.stream.synchronize()
    q0 = torch.cuda.Event(enable_timing=True)
    q1 = torch.cuda.Event(enable_timing=True)
    q0.record(sgraph.stream)
    for _ in range(nsel):
        sgraph.replay()
    q1.record(sgraph.stream)
    q1.synchronize()
    select_avg_ms = q0.elapsed_time(q1) / nsel
    attend_avg_ms = max(1e-6, (elapsed_ms / args.steps - select_avg_ms) / L)

    # ---- end to end: pinned host q', q in; outputs back to pinned host, every step
    h_slm_q = torch.empty(p.slm_q.shape, dtype=p.slm_q.dtype, pin_memory=True)
    h_slm_q.copy_(p.slm_q)
    h_q = torch.empty(p.llm_q.shape, dtype=p.llm_q.dtype, pin_memory=True)
    h_q.copy_(p.llm_q)
    h_out = torch.empty(outs.shape, dtype=outs.dtype, pin_memory=True)
    e2e_steps = max(3, min(args.steps, 200))
    if heads:
        # head sharding: the step's all-gather sits between the attends and the
        # output read, so the copies stay outside the graph, in stream order
        h2d = h_slm_q.numel() * 2 + h_q.numel() * 2
        d2h = h_out.numel() * 4
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(e2e_steps):
                p.slm_q.copy_(h_slm_q, non_blocking=True)
                p.llm_q.copy_(h_q, non_blocking=True)
                graph.replay()
                h_out.copy_(outs, non_blocking=True)
            e1.record(s)
        e1.synchronize()
    else:
        # the public API's host-I/O graph: q of layer i gates only attend i,
        # layer i's output is read back while later layers run
        hq_list = [h_q[l % resident] for l in range(L)]
        egraph = smallkv.DecodeGraph(step, p.slm_q, plan, host_io=(h_slm_q, hq_list, h_out),
                                     tier=tier)
        h2d = h_slm_q.numel() * 2 + sum(t.numel() for t in hq_list) * 2
        d2h = h_out.numel() * 4
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(egraph.stream)
        for _ in range(e2e_steps):
            egraph.replay()
        e1.record(egraph.stream)
        e1.synchronize()
        assert torch.equal(h_out, outs.cpu()), "host-I/O graph output differs from the device run"
    e2e_ms = e0.elapsed_time(e1)
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units * L * e2e_steps / (float(te.item()) / 1e3)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm, peak_kind = peaks()
    attend_bytes = bm["attend_per_layer"]
    achieved = attend_bytes / (attend_avg_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attend_dram_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        if tj.get("config") == args.config:
            traffic = tj.get("dram_bytes_per_launch")
    step_gbs = bm["step"] / (ms_per_step / 1e3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(layer_steps, 2),
        "unit": "layer-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong" if heads else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded; Fig. 2-calibrated salience, random page tables)",
        "config": {
            "workload": f"{args.config}: {cfg.description}",
            "global_batch": p.batch * units,
            "seq_len": cfg.seq_len,
            "parallelism": (f"kv-head-group sharded x{world}"
                            + (" + SLM row blocks (f3b: +1 NCCL all-gather of the selection)"
                               if slm_part else "")
                            + " (+1 NCCL all-gather of outputs per step)"
                            if heads else f"batch-sharded x{world} (no collective)"),
            "budget_K_R_M": list(cfg.budget),
            "head_map": "coherent (every SLM kv-head referenced)",
            "selection": ("f2: one split per LLM (layer, kv-group) of the summed proxy rows "
                          "(SURVEY §8(f) f2, DESIGN.md R16)" if args.variant == "f2"
                          else "per SLM row (Eq. 6, R1/R14)"
                          + ("; f4: LLM K/V pool in pinned host memory, per-group HBM hot "
                             "pools (SURVEY §8(f) f4, DESIGN.md R18)" if args.variant == "f4" else "")),
            "page_size": p.llm.page_size,
            "resident_llm_layers": resident,
            "l2": "inputs larger than L2: %.2f GB touched per step vs 126 MB L2" % (bm["step"] / 1e9),
        },
        "achieved_hbm_gbs_step": round(step_gbs, 1),
        "hbm_frac_step": round(step_gbs / hbm, 4),
        "bytes_per_step": bm["step"],
        "roofline": {
            "kernel": "attend_kernel (K3 gather-attend + fused combine)",
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": hbm,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": round(achieved / hbm, 4),
            "traffic": traffic,
            "algorithmic_bytes_per_launch": attend_bytes,
            "avg_launch_ms": round(attend_avg_ms, 5),
            "avg_launch_ms_note": "effective per-layer attend time in the PDL-pipelined step: "
                                  "(ms_per_step - select_ms) / L",
            "select_avg_ms": round(select_avg_ms, 5),
            "select_algorithmic_bytes": bm["slm_score"],
            "select_gbs": round(bm["slm_score"] / (select_avg_ms / 1e3) / 1e9, 1),
        },
        "e2e": {"value": round(e2e_value, 2), "unit": "layer-steps/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps},
        "gpu_launches": graph.kernels_per_step * args.steps,
        "clocks": clocks,
    }
    if tier is not None:
        line["f4"] = f4_report(p, cfg, graph, tier)
    if not args.no_cpu_baseline and world == 1:   # the oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(p, cfg, L, variant=args.variant)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def f4_report(p, cfg, graph, tier, steps: int = 20):
    """Host-link traffic of the tiered pool: in the steady state (same inputs
    every step) nothing is fetched after the first step; with the SLM query
    alternating between two inputs the selection drifts every step and only the
    rows that were not resident cross the host link."""
    import torch
    row_bytes = cfg.llm.head_dim * 2
    s = graph.stream
    s.synchronize()
    f0, ov0 = tier.counters()
    for _ in range(3):
        graph.replay()
    s.synchronize()
    f1, _ = tier.counters()
    g = torch.Generator(device=p.slm_q.device).manual_seed(99)
    q_a = p.slm_q.clone()
    q_b = (p.slm_q.float() + 0.1 * torch.randn(p.slm_q.shape, device=p.slm_q.device,
                                               generator=g)).to(torch.bfloat16)
    with torch.cuda.stream(s):
        p.slm_q.copy_(q_b)
    graph.replay()                                   # first drift step (outside the timing)
    s.synchronize()
    f2, _ = tier.counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(steps):
        with torch.cuda.stream(s):
            p.slm_q.copy_(q_a if i % 2 == 0 else q_b)
        graph.replay()
    e1.record(s)
    e1.synchronize()
    f3, ov = tier.counters()
    with torch.cuda.stream(s):
        p.slm_q.copy_(q_a)
    s.synchronize()
    ms = e0.elapsed_time(e1) / steps
    per = (f3 - f2) / steps
    return {"steady_rows_fetched_per_step": (f1 - f0) / 3,
            "drift": {"value": round(cfg.llm.layers / (ms / 1e3), 2), "unit": "layer-steps/s",
                      "ms_per_step": round(ms, 4), "rows_fetched_per_step": per,
                      "host_link_bytes_per_step": int(per * row_bytes),
                      "host_link_gbs": round(per * row_bytes / (ms / 1e3) / 1e9, 2),
                      "note": "SLM query alternating between two inputs each step"},
            "capacity_overflows": ov,
            "hot_pool_bytes": int(tier.hot_k.numel() * 4),
            "host_pool_bytes": int(p.llm.k.numel() * 4)}


def cpu_baseline(p, cfg, L, target_s: float = 12.0, variant: str = "default"):
    """Time the oracle, as it stands, on a bounded sample of the same step:
    every sequence of the batch, the select for every SLM row the step uses,
    and the attend of as many LLM layers as fit in ~target_s seconds; the
    per-layer attend time is extrapolated to all L layers."""
    import dataclasses
    import oracle
    from tests import parity

    def cpu_layer(slot):
        return dataclasses.replace(
            p, llm_q=p.llm_q[slot:slot + 1].contiguous(),
            llm=dataclasses.replace(p.llm, k=p.llm.k[slot:slot + 1].contiguous(),
                                    v=p.llm.v[slot:slot + 1].contiguous()),
            llm_layer_ids=[p.llm_layer_ids[slot]]).to("cpu")

    base = cpu_layer(0)
    slm_v, _ = parity.views(base)
    rows = oracle.image_rows(base.head_map)
    t0 = time.perf_counter()
    sel = parity.oracle_select(base, rows=rows, slm_view=slm_v)
    t_sel = time.perf_counter() - t0
    t_layers = []
    slot = 0
    while slot < p.llm.num_layers:
        sub = base if slot == 0 else cpu_layer(slot)
        _, llm_v = parity.views(sub)
        t1 = time.perf_counter()
        n_slm = cfg.slm.layers * cfg.slm.q_heads
        if variant == "f2":
            gsel = oracle.select_group(sub.llm_layer_ids[0], cfg.llm.q_heads, cfg.llm.kv_heads,
                                       sub.head_map, sel, sub.seq_lens, sub.k_crit, sub.n_recent,
                                       sub.k_marg, sub.max_crit, sub.max_marg, n_slm)
            oracle.attend_group(sub.llm_layer_ids[0], 0, sub.llm_q[0], llm_v, sub.seq_lens,
                                sub.head_map, sel, gsel, n_slm)
        else:
            oracle.attend(sub.llm_layer_ids[0], 0, sub.llm_q[0], llm_v, sub.seq_lens,
                          sub.head_map, sel, n_slm)
        t_layers.append(time.perf_counter() - t1)
        slot += 1
        if t_sel + sum(t_layers) >= target_s:
            break
    t_step = t_sel + L * (sum(t_layers) / len(t_layers))
    return {"value": round(L / t_step, 4), "unit": "layer-steps/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": (f"all {p.batch} sequences: select over all {len(rows)} mapped SLM rows "
                       f"({t_sel:.2f} s) + attend of {len(t_layers)} of {L} LLM layers "
                       f"({sum(t_layers):.2f} s), per-layer time extrapolated to {L} layers"),
            "measured_s": round(t_sel + sum(t_layers), 3)}


def run_reference(args, world, rank, local):
    """The oracle as the reference arm (rank 0 only), same metric and config."""
    if rank != 0:
        return
    import torch
    import oracle
    import smallkv_synth as synth
    from tests import parity

    oracle.build()
    cfg = synth.CONFIGS[args.config]
    L = cfg.llm.layers
    n_seqs = args.cpu_seqs
    p = synth.make_problem(cfg, seed=0, device="cpu", batch=n_seqs, llm_layers=[0])
    slm_v, llm_v = parity.views(p)
    rows = oracle.image_rows(p.head_map)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sel = parity.oracle_select(p, rows=rows, slm_view=slm_v)
        t1 = time.perf_counter()
        oracle.attend(0, 0, p.llm_q[0], llm_v, p.seq_lens, p.head_map, sel,
                      cfg.slm.layers * cfg.slm.q_heads)
        t2 = time.perf_counter()
        if it >= args.warmup:
            times.append((t1 - t0) + L * (t2 - t1))
    t_step = statistics.mean(times) * cfg.batch / n_seqs
    value = L / t_step
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "layer-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.description}", "global_batch": cfg.batch,
                   "seq_len": cfg.seq_len, "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": round(value, 4), "unit": "layer-steps/s",
                         "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": (f"each step: {n_seqs} of {cfg.batch} sequences, select over "
                                    f"all {len(rows)} mapped SLM rows + 1 LLM layer attend, "
                                    f"extrapolated to {L} layers x {cfg.batch} sequences")},
        "e2e": {"value": round(value, 4), "unit": "layer-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="qwen7b")
    ap.add_argument("--variant", choices=["default", "f2", "f4"], default="default",
                    help="f2: per-KV-group shared selection (SURVEY §8(f) f2, DESIGN.md R16); "
                         "f4: host-tiered KV pool (SURVEY §8(f) f4, DESIGN.md R18)")
    ap.add_argument("--shard", choices=["batch", "heads", "heads-slm"], default="batch",
                    help="N>1 partition: sequences (weak scaling) or LLM kv-head groups")
    ap.add_argument("--cpu-seqs", type=int, default=4,
                    help="sequences per step of the --impl reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="profiling mode: only warm-up + timed replays (for ncu launch lists)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
