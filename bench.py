#!/usr/bin/env python
"""Benchmark of the SmallKV decode hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config qwen7b] [--shard batch|heads|heads-slm]
                    [--tau T] [--seq-len N] [--emulate-world G] [--decode-run]

A step = one pass of the whole hot path over one batch: smallkv_select over
all SLM layers (K1 score + K2 split) and one smallkv_attend per LLM layer
(K3 gather-attend with the fused combine), captured in one CUDA graph.
Metric (BASELINE.json): decode-attention layer-steps/s (= L LLM layers per
step, for the whole global batch) and achieved HBM GB/s over the algorithmic
bytes of DESIGN.md §7.  Default workload: BASELINE.json configs[1]
(Qwen2.5-7B + Qwen2.5-0.5B, ctx 4096, batch 32).

N > 1 (torchrun, one rank per GPU), strong scaling of the config's global
batch: `--shard batch` (default) gives rank r the sequences
batch_shard(B, N, r), no data-path collective; `--shard heads` gives it LLM
kv-groups [r*H_kv/N, (r+1)*H_kv/N) of every sequence and all-gathers the
per-head outputs once per step (NCCL); `--shard heads-slm` (f3b) also splits
the SLM rows and all-gathers the selection.  The step time is the max over
ranks (device clock, CUDA events).

`--emulate-world G` (1 GPU): time rank 0's exact workload of a G-rank job and
project the job's throughput and scaling efficiency from it (plus an NCCL
cost model for the head-split exchanges); the line is labelled "emulated".
`--decode-run`: the long-generation setting of BASELINE configs[4] — the
same graph replayed at growing context n (budgets from tau at each n).

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


def workload(args):
    """The config with the command line's overrides (--tau, --seq-len)."""
    import dataclasses
    import smallkv_synth as synth
    cfg = synth.CONFIGS[args.config]
    if args.seq_len:
        cfg = dataclasses.replace(cfg, seq_len=args.seq_len)
    tau = args.tau if args.tau else (cfg.tau if args.seq_len else None)
    if tau:
        n = cfg.seq_len
        if args.config == "llama8b" and n == 32768 and tau in synth.LLAMA8B_SWEEP:
            bud = synth.LLAMA8B_SWEEP[tau]
        else:   # P:235 2:1:2 split (R6)
            bud = (int(tau * n / 2 + 1e-9), int(tau * n / 4 + 1e-9), int(tau * n / 2 + 1e-9))
        cfg = dataclasses.replace(cfg, budget=bud, tau=tau)
    return cfg


def f4_capacity(cfg) -> int:
    """f4 hot-pool slots per group: the largest list R' + (#distinct SLM rows of
    the group) * (K'+M') under the config's head map and budgets."""
    import smallkv_synth as synth
    L, H, Hkv = cfg.llm.layers, cfg.llm.q_heads, cfg.llm.kv_heads
    hm = synth.head_map_coherent(cfg.llm, cfg.slm).view(L, Hkv, H // Hkv)
    rows_max = max(len(set(hm[l, g].tolist())) for l in range(L) for g in range(Hkv))
    K, R, M = cfg.budget
    return -(-(R + rows_max * (K + M)) // 4) * 4


def f4_device_bytes(cfg, B: int) -> int:
    """HBM the f4 hot pools (K and V) and tier state take."""
    cap = f4_capacity(cfg)
    groups = cfg.llm.layers * B * cfg.llm.kv_heads
    return groups * cap * cfg.llm.head_dim * 2 * 2 + groups * (cfg.seq_len * 4 + cap * 21)


def build_problem(cfg, rank: int, world: int, shard: str, device, reserve: int = 0,
                  max_resident: int = 0):
    """Rank `rank`'s inputs of a `world`-rank job over the config's GLOBAL batch
    (strong scaling).  batch sharding: the sequences batch_shard(B, world, rank)
    (drawn with seed = rank; every rank holds both models' caches of its own
    sequences).  head sharding: the whole batch (seed 0) with the LLM side
    restricted to this rank's kv-groups."""
    import dataclasses
    import torch
    import smallkv_synth as synth
    from paper_2508_02751_b200 import dist as pdist
    heads = shard in ("heads", "heads-slm") and world > 1
    if heads and cfg.llm.kv_heads % world:
        raise SystemExit(f"{cfg.llm.kv_heads} LLM kv-heads do not split over {world} ranks")
    B = cfg.batch if heads else len(pdist.batch_shard(cfg.batch, world, rank))
    kv_share = cfg.llm.kv_heads // world if heads else cfg.llm.kv_heads
    # resident LLM layers: all when they fit, else a rotating subset (each slice >> L2)
    per_layer = B * kv_share * cfg.seq_len * cfg.llm.head_dim * 2 * 2
    free = torch.cuda.mem_get_info(device)[0]
    slm_bytes = cfg.slm.layers * B * cfg.slm.kv_heads * cfg.seq_len * cfg.slm.head_dim * 2
    budget = int(0.8 * free) - slm_bytes - (4 << 30) - reserve
    if heads:   # the full LLM pool is generated once, then sliced (a copy of the slice)
        budget = budget * kv_share // (cfg.llm.kv_heads + kv_share)
    resident = max(1, min(cfg.llm.layers, budget // per_layer))
    if max_resident:
        resident = min(resident, max_resident)
    p = synth.make_problem(cfg, seed=0 if heads else rank, device=device, batch=B,
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


# NCCL over NVLink 5 (B200_PROFILING.md: 8-rank all-reduce bus bandwidth 725 GB/s,
# peer copy 770 GB/s per direction); per-call latency of a small all-gather on
# one node, an estimate (no multi-GPU box was available to measure it)
NCCL_BW_GBS = 725.0
NCCL_LAT_US = 15.0


def allgather_ms(total_bytes: int, world: int, calls: int = 1) -> float:
    """Ring/NVLS all-gather time model: each rank receives (world-1)/world of
    the gathered tensor; `calls` collective launches."""
    if world <= 1:
        return 0.0
    return calls * NCCL_LAT_US / 1e3 + total_bytes * (world - 1) / world / (NCCL_BW_GBS * 1e9) * 1e3


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    emulate = args.emulate_world > 1 and world == 1
    jw, jr = (args.emulate_world, 0) if emulate else (world, rank)   # the job's world / this rank
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    from paper_2508_02751_b200 import build as kbuild
    if rank == 0:
        kbuild.build()
    if world > 1:
        dist.barrier()
    from paper_2508_02751_b200 import bytes_model, smallkv
    from paper_2508_02751_b200 import dist as pdist

    cfg = workload(args)
    heads = args.shard in ("heads", "heads-slm") and jw > 1
    slm_part = args.shard == "heads-slm" and jw > 1
    if args.variant == "f4":
        # the hot pools and tier state stay in HBM; the host copy of the resident
        # layer slots must fit pinned host memory (half of it at most)
        import psutil
        B0 = len(pdist.batch_shard(cfg.batch, jw, jr))
        per_layer = B0 * cfg.llm.kv_heads * cfg.seq_len * cfg.llm.head_dim * 2 * 2
        p, resident = build_problem(cfg, jr, jw, args.shard, device, reserve=f4_device_bytes(cfg, B0),
                                    max_resident=max(1, psutil.virtual_memory().total // 2 // per_layer))
    else:
        p, resident = build_problem(cfg, jr, jw, args.shard, device)
    L = cfg.llm.layers
    tier = None
    if args.variant == "f4":
        # host-tiered pool: the LLM K/V in pinned host memory,
        # each group's needed rows in an HBM hot pool refreshed per layer.  The
        # host pool holds the problem's resident layer slots (LLM layer l reads
        # slot l mod resident, as the HBM path's rotation); the hot pool has a
        # slot per LLM layer.
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
        assert cap <= f4_capacity(cfg), (cap, f4_capacity(cfg))
        per_layer = args.f4_refresh == "per-layer"
        tier = smallkv.TieredKV(step, host_k, host_v, capacity=cap, use_plan=not per_layer,
                                per_layer=per_layer)
    else:
        step = smallkv.from_problem(p, variant=args.variant)
    H_loc, d = p.cfg.llm.q_heads, cfg.llm.head_dim
    outs = torch.empty(L, p.batch, H_loc, d, dtype=torch.float32, device=device)
    plan = [(l, l % resident, p.llm_q[l % resident], outs[l]) for l in range(L)]
    graph = smallkv.DecodeGraph(step, p.slm_q, plan, timing=False, tier=tier)
    n_slm = cfg.slm.layers * cfg.slm.q_heads
    comm_ms_model = 0.0       # emulated exchange time per step (NCCL cost model)
    exch_bytes = 0
    if slm_part:
        # f3b: this rank scores / splits only its block of SLM rows, the blocks
        # are all-gathered (NCCL), then the plan and this rank's kv-group attends
        # run on the exchanged selection; the step runs eagerly (collective inside).
        # Emulated: the other ranks' rows come from one untimed full selection.
        j0, j1 = pdist.slm_row_block(n_slm, jw, jr)
        shm = pdist.select_head_map(p.full_head_map.to(device), j0, j1)
        exch_bytes = pdist.exchange_bytes(step.out, n_slm, jw)
        if emulate:
            step.select(p.slm_q, plan=False)
            torch.cuda.synchronize()
            comm_ms_model += len(pdist.SELECTION_FIELDS) * NCCL_LAT_US / 1e3 + \
                exch_bytes / (NCCL_BW_GBS * 1e9) * 1e3

        def replay_f3b():
            with torch.cuda.stream(graph.stream):
                step.select(p.slm_q, select_head_map=shm, plan=False)
                if not emulate:
                    pdist.exchange_selection(step.out, n_slm)
                step.plan()
                for i, (layer, slot, q, out) in enumerate(plan):
                    step.attend(layer, slot, q, out, overlap_prologue=i > 0)
        graph.replay = replay_f3b
    gathered = None
    gather_bytes = L * p.batch * cfg.llm.q_heads * d * 4   # the [L, B, H, d] fp32 outputs
    if heads:
        # the exchange step of head sharding: all-gather every layer's per-head
        # outputs once per step into a rank-major [world, L, B, H/w, d] buffer
        # (head h = rank * H/w + local head), NCCL over NVLink
        if emulate:
            comm_ms_model += allgather_ms(gather_bytes, jw)
        else:
            gathered = torch.empty((world,) + tuple(outs.shape), dtype=outs.dtype, device=device)
            inner = graph.replay

            def replay_and_gather():
                inner()
                with torch.cuda.stream(graph.stream):
                    dist.all_gather_into_tensor(gathered, outs)
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
    if args.decode_run:
        return decode_run(args, p, cfg, graph, step, L, rank, world)
    sgraph = smallkv.DecodeGraph(step, p.slm_q, [], timing=False)   # select only
    # isolated attend launches: CUDA events between the calls (no PDL overlap)
    tgraph = smallkv.DecodeGraph(step, p.slm_q, plan, timing=True) if not slm_part else None
    # serialised launches: the same step with no attend overlapping the previous
    # one (each waits for its predecessor before it reads anything)
    igraph = (smallkv.DecodeGraph(step, p.slm_q, plan, timing=False, overlap=False)
              if not slm_part and tier is None else None)

    seq = [int(x) for x in p.seq_lens.cpu()]
    buds = list(zip(p.k_crit.cpu().tolist(), p.n_recent.cpu().tolist(), p.k_marg.cpu().tolist()))
    bm = bytes_model.step_bytes_coherent(p.cfg, seq, buds, L)
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
    # one layer-step = one LLM layer of the whole GLOBAL batch (all heads)
    layer_steps = L * args.steps / (max_ms / 1e3)

    # ---- per-kernel durations (CUDA events on the graphs' streams):
    # select alone (back-to-back replays); attend isolated (events between the
    # launches, so no cross-layer PDL overlap) and pipelined-effective
    # ((step - select) / L, credits the overlap of consecutive layers)
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
    step_local_ms = elapsed_ms / args.steps
    attend_pipe_ms = max(1e-6, (step_local_ms - select_avg_ms) / L)
    attend_iso_ms = None
    attend_ev_ms = None
    if tgraph is not None:
        samples = []
        for _ in range(max(5, min(args.steps, 50))):
            tgraph.replay()
            tgraph.stream.synchronize()
            samples.extend(tgraph.segment_ms()[1])
        attend_ev_ms = statistics.median(samples)
    if igraph is not None:
        for _ in range(3):
            igraph.replay()
        igraph.stream.synchronize()
        i0 = torch.cuda.Event(enable_timing=True)
        i1 = torch.cuda.Event(enable_timing=True)
        i0.record(igraph.stream)
        for _ in range(nsel):
            igraph.replay()
        i1.record(igraph.stream)
        i1.synchronize()
        attend_iso_ms = max(1e-6, (i0.elapsed_time(i1) / nsel - select_avg_ms) / L)
    elif attend_ev_ms is not None:
        attend_iso_ms = attend_ev_ms

    # ---- end to end: pinned host q', q in; outputs back to pinned host, every step
    e2e = None
    if not emulate:
        e2e = end_to_end(args, p, graph, step, plan, outs, gathered, heads, resident, tier, L,
                         world, device, barrier)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm, peak_kind = peaks()
    attend_bytes = bm["attend_per_layer"]
    launch_ms = attend_iso_ms if attend_iso_ms is not None else attend_pipe_ms
    achieved = attend_bytes / (launch_ms / 1e3) / 1e9
    achieved_pipe = attend_bytes / (attend_pipe_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        if tj.get("budget") in (None, list(p.cfg.budget)) and not emulate:
            traffic = tj.get("attend_dram_bytes_per_launch")
    step_gbs = bm["step"] / (ms_per_step / 1e3) / 1e9
    par = (f"kv-head-group sharded x{jw}"
           + (" + SLM row blocks (f3b: +1 NCCL all-gather of the selection)" if slm_part else "")
           + " (+1 NCCL all-gather of outputs per step)"
           if heads else f"batch-sharded x{jw} over the global batch (no collective)")
    line = {
        "metric": METRIC,
        "value": round(layer_steps, 2),
        "unit": "layer-steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded; Fig. 2-calibrated salience, random page tables)",
        "config": {
            "workload": f"{args.config}: {cfg.description}",
            "global_batch": cfg.batch,
            "local_batch": p.batch,
            "seq_len": cfg.seq_len,
            "parallelism": par,
            "budget_K_R_M": list(p.cfg.budget),
            "tau": p.cfg.tau,
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
            "avg_launch_ms": round(launch_ms, 5),
            "avg_launch_ms_note": ("serialised launches: (a graph of select + L attends, none "
                                   "overlapping its predecessor) - select, per layer"
                                   if igraph is not None else
                                   "median isolated launch: CUDA events between the attend "
                                   "launches of a timing graph (no cross-layer PDL overlap)"
                                   if attend_iso_ms is not None else
                                   "pipelined-effective: (ms_per_step - select_ms) / L"),
            "event_bracketed_launch_ms": None if attend_ev_ms is None else round(attend_ev_ms, 5),
            "achieved_pipelined": round(achieved_pipe, 1),
            "frac_pipelined": round(achieved_pipe / hbm, 4),
            "pipelined_ms_per_layer": round(attend_pipe_ms, 5),
            "pipelined_note": "(ms_per_step - select_ms) / L inside the PDL-chained step "
                              "(consecutive layers overlap prologue and tail): derived",
            "select_avg_ms": round(select_avg_ms, 5),
            "select_algorithmic_bytes": bm["slm_score"],
            "select_gbs": round(bm["slm_score"] / (select_avg_ms / 1e3) / 1e9, 1),
        },
        "e2e": e2e,
        "gpu_launches": graph.kernels_per_step * args.steps,
        "clocks": clocks,
    }
    if emulate:
        rank_ms = step_local_ms
        proj_ms = rank_ms + comm_ms_model
        line["emulated"] = {
            "world": jw, "rank": jr, "mode": args.shard,
            "note": ("one B200 runs rank 0's exact workload of a %d-rank job; ranks are "
                     "symmetric (equal shards), so the job's step time is projected as rank 0's "
                     "device time plus the modelled NCCL exchange" % jw),
            "rank_ms_per_step": round(rank_ms, 5),
            "comm_ms_model": round(comm_ms_model, 5),
            "comm_model": {"allgather_bytes_per_step": gather_bytes if heads else 0,
                           "selection_exchange_bytes_per_rank": exch_bytes,
                           "nvlink_gbs": NCCL_BW_GBS, "latency_us_per_call": NCCL_LAT_US},
            "projected_ms_per_step": round(proj_ms, 5),
            "projected_value": round(L / (proj_ms / 1e3), 2),
        }
        line["value"] = line["emulated"]["projected_value"]
        line["ms_per_step"] = round(proj_ms, 5)
        line["n_gpus"] = 1
        line["data"] += "; EMULATED %d-rank job on 1 GPU" % jw
    if tier is not None:
        line["f4"] = f4_report(p, cfg, graph, tier)
    if not args.no_cpu_baseline and world == 1 and not emulate:   # rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(p, cfg, L, variant=args.variant)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def end_to_end(args, p, graph, step, plan, outs, gathered, heads, resident, tier, L, world,
               device, barrier):
    """The same metric through the public API with host buffers: pinned q', q in
    and every layer's output (head split: the gathered outputs) out, inside the
    timed region, every step."""
    import torch
    import torch.distributed as dist
    from paper_2508_02751_b200 import smallkv
    h_slm_q = torch.empty(p.slm_q.shape, dtype=p.slm_q.dtype, pin_memory=True)
    h_slm_q.copy_(p.slm_q)
    h_q = torch.empty(p.llm_q.shape, dtype=p.llm_q.dtype, pin_memory=True)
    h_q.copy_(p.llm_q)
    e2e_steps = max(3, min(args.steps, 200))
    if heads:
        # head sharding: the step's all-gather sits between the attends and the
        # output read, so the copies stay outside the graph, in stream order;
        # the read-back is the gathered [world, L, B, H/w, d] tensor
        h_out = torch.empty(gathered.shape, dtype=gathered.dtype, pin_memory=True)
        h2d = h_slm_q.numel() * 2 + h_q.numel() * 2
        d2h = h_out.numel() * 4
        s = graph.stream
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
                h_out.copy_(gathered, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        # the gathered tensor holds this rank's heads at its rank slot
        assert torch.equal(h_out[dist.get_rank()], outs.cpu()), "gathered outputs differ"
    else:
        # the public API's host-I/O graph: q of layer i gates only attend i,
        # layer i's output is read back while later layers run
        h_out = torch.empty(outs.shape, dtype=outs.dtype, pin_memory=True)
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
    value = L * e2e_steps / (float(te.item()) / 1e3)
    return {"value": round(value, 2), "unit": "layer-steps/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": e2e_steps}


def decode_run(args, p, cfg, graph, step, L, rank, world):
    """BASELINE configs[4]'s long generation: the pools hold the final context
    (cfg.seq_len); the step graph is replayed with every sequence at growing n
    (8193 -> seq_len) and tau budgets at that n (R6), i.e. per-step
    reselection over a growing cache (Alg. 1 decode loop).  The K/V
    of the positions that the decode appends are pre-drawn."""
    import torch
    from paper_2508_02751_b200 import bytes_model
    hbm, _ = peaks()
    tau = cfg.tau or 0.2
    n0 = args.decode_start
    points = sorted(set([n0] + [n0 + (cfg.seq_len - n0) * k // 4 for k in range(1, 5)]))
    res = []
    s = graph.stream
    for n in points:
        bud = (int(tau * n / 2 + 1e-9), int(tau * n / 4 + 1e-9), int(tau * n / 2 + 1e-9))
        with torch.cuda.stream(s):
            p.seq_lens.fill_(n)
            p.k_crit.fill_(min(bud[0], p.max_crit))
            p.n_recent.fill_(bud[1])
            p.k_marg.fill_(min(bud[2], p.max_marg))
        for _ in range(args.warmup):
            graph.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            graph.replay()
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        bm = bytes_model.step_bytes_coherent(cfg, [n] * p.batch, [bud] * p.batch, L)
        res.append({"n": n, "budget_K_R_M": list(bud), "ms_per_step": round(ms, 4),
                    "value": round(L / (ms / 1e3), 2),
                    "step_gbs": round(bm["step"] / (ms / 1e3) / 1e9, 1),
                    "hbm_frac_step": round(bm["step"] / (ms / 1e3) / 1e9 / hbm, 4)})
    if rank == 0:
        print(json.dumps({"metric": METRIC, "decode_run": res, "unit": "layer-steps/s",
                          "config": {"workload": f"{args.config}: {cfg.description}",
                                     "global_batch": cfg.batch, "tau": tau,
                                     "max_seq_len": cfg.seq_len,
                                     "resident_llm_layers": p.llm.num_layers},
                          "steps_per_point": args.steps}), flush=True)


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
    # the host link's copy peak on this box: pinned host -> device, 1 GiB
    hb = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    db = torch.empty(1 << 30, dtype=torch.uint8, device=p.slm_q.device)
    db.copy_(hb, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(3):
        db.copy_(hb, non_blocking=True)
    c1.record()
    c1.synchronize()
    link_peak = 3 * (1 << 30) / (c0.elapsed_time(c1) / 1e3) / 1e9
    del hb, db
    return {"steady_rows_fetched_per_step": (f1 - f0) / 3,
            "refresh": "per-layer (side stream, overlaps the attends)" if tier.per_layer
                       else "all layers in one launch after select",
            "host_link_peak_gbs": round(link_peak, 2),
            "drift": {"value": round(cfg.llm.layers / (ms / 1e3), 2), "unit": "layer-steps/s",
                      "ms_per_step": round(ms, 4), "rows_fetched_per_step": per,
                      "host_link_bytes_per_step": int(per * row_bytes),
                      "host_link_gbs": round(per * row_bytes / (ms / 1e3) / 1e9, 2),
                      "host_link_frac": round(per * row_bytes / (ms / 1e3) / 1e9 / link_peak, 3),
                      "note": "SLM query alternating between two inputs each step"},
            "capacity_overflows": ov,
            "hot_pool_bytes": int(tier.hot_k.numel() * 4),
            "host_pool_bytes": int(p.llm.k.numel() * 4)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
            "cpu_model": cpu_model(), "kind": "oracle",
            "sample": (f"all {p.batch} sequences: select over all {len(rows)} mapped SLM rows "
                       f"({t_sel:.2f} s) + attend of {len(t_layers)} of {L} LLM layers "
                       f"({sum(t_layers):.2f} s), per-layer time extrapolated to {L} layers"),
            "measured_s": round(t_sel + sum(t_layers), 3)}


def run_reference(args, world, rank, local):
    """The oracle as the reference arm (rank 0 only), same metric and config.

    Config 2 and smaller: every step is the WHOLE step on the host cores — the
    split of every mapped SLM row for every sequence plus the attend of all L
    LLM layers (their K/V rotated through one resident layer, as the GPU arm
    rotates through its resident layers) — so ms_per_step is measured, not
    extrapolated.  Larger configs: each step is a bounded sample (--cpu-seqs
    sequences, one LLM layer) and the value is extrapolated to the workload;
    ms_per_step is then the sample's measured time."""
    if rank != 0:
        return
    import oracle
    import smallkv_synth as synth
    from tests import parity

    oracle.build()
    cfg = workload(args)
    L = cfg.llm.layers
    full = cfg.batch * cfg.seq_len <= 32 * 4096
    n_seqs = cfg.batch if full else min(args.cpu_seqs, cfg.batch)
    n_att = L if full else 1
    p = synth.make_problem(cfg, seed=0, device="cpu", batch=n_seqs, llm_layers=[0])
    slm_v, llm_v = parity.views(p)
    rows = oracle.image_rows(p.head_map)
    n_slm = cfg.slm.layers * cfg.slm.q_heads
    times, t_sel, t_att = [], [], []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sel = parity.oracle_select(p, rows=rows, slm_view=slm_v)
        t1 = time.perf_counter()
        for layer in range(n_att):
            # LLM layer `layer` (head map row), K/V of the resident slot 0
            oracle.attend(layer, 0, p.llm_q[0], llm_v, p.seq_lens, p.head_map, sel, n_slm)
        t2 = time.perf_counter()
        if it >= args.warmup:
            times.append(t2 - t0)
            t_sel.append(t1 - t0)
            t_att.append((t2 - t1) / n_att)
    ms_sample = statistics.mean(times) * 1e3
    t_step = (statistics.mean(t_sel) + L * statistics.mean(t_att)) * cfg.batch / n_seqs
    value = L / t_step
    sample = (f"each step: all {cfg.batch} sequences, select over all {len(rows)} mapped SLM rows "
              f"+ attend of all {L} LLM layers (K/V rotated through one resident layer)" if full else
              f"each step: {n_seqs} of {cfg.batch} sequences, select over all {len(rows)} mapped "
              f"SLM rows + 1 LLM layer attend; value extrapolated to {L} layers x {cfg.batch} "
              f"sequences ({t_step * 1e3:.1f} ms per full step)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "layer-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_sample, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.description}", "global_batch": cfg.batch,
                   "seq_len": cfg.seq_len, "parallelism": "host cores (OpenMP)",
                   "budget_K_R_M": list(cfg.budget)},
        "cpu_baseline": {"value": round(value, 4), "unit": "layer-steps/s",
                         "cores": oracle.num_threads(), "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "layer-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not full:
        line["extrapolated_ms_per_step"] = round(t_step * 1e3, 3)
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
    ap.add_argument("--f4-refresh", choices=["per-layer", "all"], default="all",
                    help="f4: refresh layer l+1's hot pool on a side stream during attend l "
                         "(per-layer), or every layer in one launch after select (all)")
    ap.add_argument("--shard", choices=["batch", "heads", "heads-slm"], default="batch",
                    help="N>1 partition of the global batch: sequences or LLM kv-head groups")
    ap.add_argument("--emulate-world", type=int, default=1,
                    help="1 GPU: time rank 0's workload of a G-rank job, project the job")
    ap.add_argument("--tau", type=float, default=None,
                    help="budget fraction (P:235 2:1:2 split; llama8b sweep 0.05-0.5)")
    ap.add_argument("--seq-len", type=int, default=None, help="context length override")
    ap.add_argument("--decode-run", action="store_true",
                    help="replay the step at growing n (--decode-start .. seq_len)")
    ap.add_argument("--decode-start", type=int, default=8193)
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
