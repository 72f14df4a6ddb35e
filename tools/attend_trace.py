"""Per-CTA globaltimer trace of one decode step's attend launches (diagnostic).

Builds libsmallkv with -DSKV_TRACE into exp/libs/trace.so (thread 0 of every
attend CTA stores %globaltimer at fixed points, gather_attend.cu SKV_T), runs
bench.py's workload through a DecodeGraph, replays one traced step and prints,
per layer and summed over the step: launch-to-launch spacing, the prologue
(start -> batch 0 staged -> first tile), the main loop, CTA-synchronous batch
staging, the merge, and the tail (slowest CTA vs median CTA).

    python tools/attend_trace.py --config qwen7b [--json out.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SLOTS = 16
LIB = os.path.join(ROOT, "exp", "libs", "trace.so")


def build_trace_lib() -> str:
    from paper_2508_02751_b200 import build as b
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cmd = [b.NVCC] + b.FLAGS + ["-DSKV_TRACE", "-o", LIB] + b.SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        raise SystemExit("trace build failed")
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen7b")
    ap.add_argument("--variant", default="default")
    ap.add_argument("--no-build", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--emulate-world", type=int, default=1,
                    help="trace rank 0's batch shard of a G-rank job (small batches)")
    args = ap.parse_args()
    if not args.no_build:
        build_trace_lib()
    os.environ["SMALLKV_LIB"] = LIB
    import numpy as np
    import torch
    import bench
    from paper_2508_02751_b200 import smallkv

    ns = argparse.Namespace(config=args.config, tau=None, seq_len=None)
    cfg = bench.workload(ns)
    dev = torch.device("cuda:0")
    p, resident = bench.build_problem(cfg, 0, args.emulate_world, "batch", dev)
    L = cfg.llm.layers
    step = smallkv.from_problem(p, variant=args.variant)
    outs = torch.empty(L, p.batch, p.cfg.llm.q_heads, cfg.llm.head_dim, dtype=torch.float32, device=dev)
    plan = [(l, l % resident, p.llm_q[l % resident], outs[l]) for l in range(L)]
    graph = smallkv.DecodeGraph(step, p.slm_q, plan, timing=False)
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    buf = torch.zeros(L * 4096 * SLOTS, dtype=torch.int64, device=dev)
    lib = smallkv.load()
    lib.skv_debug_set_trace.argtypes = [ctypes.c_void_p]
    assert lib.skv_debug_set_trace(buf.data_ptr()) == 0
    graph.replay()
    torch.cuda.synchronize()
    assert lib.skv_debug_set_trace(None) == 0
    tr = buf.view(L, 4096, SLOTS).cpu().numpy()
    rows = []
    prev_end = None
    t_origin = None
    for l in range(L):
        r = tr[l]
        live = r[:, 7] > 0
        r = r[live]
        if len(r) == 0:
            continue
        t0 = r[:, 7].min()
        if t_origin is None:
            t_origin = t0
        end_col = np.where(r[:, 5] > 0, r[:, 5], r[:, 4])
        end = np.maximum(end_col, r[:, 6]).max()
        rel = lambda c: float(np.median(r[:, c] - t0)) / 1e3   # noqa: E731  (us)
        rows.append({
            "layer": l, "ctas": int(len(r)),
            "start_spread_us": float(r[:, 7].max() - t0) / 1e3,
            "gap_from_prev_us": None if prev_end is None else float(t0 - prev_end) / 1e3,
            "griddep_us": rel(0), "layout_us": rel(1), "batch0_us": rel(2),
            "loop_end_us": rel(4), "merge_end_us": float(np.median(end_col - t0)) / 1e3,
            "last_end_us": float(end - t0) / 1e3,
            "sync_stage_us": float(np.median(r[:, 12])) / 1e3,
            "batches": float(np.median(r[:, 13])), "entries": float(np.median(r[:, 10])),
            "entries_min": int(r[:, 10].min()), "entries_max": int(r[:, 10].max()),
            "loop_us_min": float((r[:, 4] - r[:, 0]).min()) / 1e3,
            "loop_us_med": float(np.median(r[:, 4] - r[:, 0])) / 1e3,
            "loop_us_max": float((r[:, 4] - r[:, 0]).max()) / 1e3,
            # per-CTA streaming rate (entries per us) spread: imbalance of bytes vs of rate
            "rate_min": float((r[:, 10] / np.maximum(r[:, 4] - r[:, 2], 1) * 1e3).min()),
            "rate_max": float((r[:, 10] / np.maximum(r[:, 4] - r[:, 2], 1) * 1e3).max()),
        })
        prev_end = end
    keys = ["griddep_us", "layout_us", "batch0_us", "loop_end_us", "merge_end_us", "last_end_us",
            "sync_stage_us", "start_spread_us", "entries_min", "entries", "entries_max",
            "loop_us_min", "loop_us_med", "loop_us_max", "rate_min", "rate_max"]
    summ = {k: float(np.mean([x[k] for x in rows])) for k in keys}
    gaps = [x["gap_from_prev_us"] for x in rows if x["gap_from_prev_us"] is not None]
    summ["gap_from_prev_us"] = float(np.mean(gaps)) if gaps else 0.0
    summ["step_attend_span_us"] = float(prev_end - t_origin) / 1e3
    print("layer  ctas  gap   dep   lay   b0    loop   merge  last   sstage  batches entries")
    for x in rows:
        print(f"{x['layer']:5d} {x['ctas']:5d} {x['gap_from_prev_us'] or 0:5.2f} {x['griddep_us']:5.2f} "
              f"{x['layout_us']:5.2f} {x['batch0_us']:5.2f} {x['loop_end_us']:6.2f} {x['merge_end_us']:6.2f} "
              f"{x['last_end_us']:6.2f} {x['sync_stage_us']:6.2f} {x['batches']:5.1f} {x['entries']:7.0f}")
    print(json.dumps({"config": args.config, "mean_per_layer": summ}))
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"config": args.config, "mean_per_layer": summ, "layers": rows}, f, indent=1)


if __name__ == "__main__":
    main()
