"""Single-GPU emulation of the multi-GPU scaling curve (one B200 per call).

    python tools/emulate_scaling.py --config qwen72b --out profiles/r02_emulated_scaling.json

For g in {1, 2, 4, 8} and each partition (batch, heads, heads-slm) it runs
`bench.py --emulate-world g` — rank 0's exact workload of a g-rank job over
the config's GLOBAL batch, timed on this GPU — and collects the projected job
throughput (rank 0's device step time + the modelled NCCL exchange) and the
strong-scaling efficiency eff(g) = value(g) / (g * value(1)).
Everything in the output is labelled as emulated: no multi-GPU node was used.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, g, shard):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", args.config,
           "--steps", str(args.steps), "--warmup", str(args.warmup), "--no-cpu-baseline",
           "--shard", shard, "--emulate-world", str(g)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=args.timeout)
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"error": (r.stderr or r.stdout)[-800:]}
    return json.loads(lines[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen72b")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--timeout", type=int, default=900)
    ap.add_argument("--modes", default="batch,heads,heads-slm")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    worlds = [int(x) for x in args.worlds.split(",")]
    base = run(args, 1, "batch")
    v1 = base.get("value")
    out = {"config": args.config, "emulated": True,
           "note": ("single-GPU emulation: each entry times rank 0's exact workload of a g-rank "
                    "job over the config's global batch on one B200 and adds a modelled NCCL "
                    "exchange (bench.py allgather_ms); eff(g) = value(g) / (g * value(1))"),
           "g1": {"value": v1, "ms_per_step": base.get("ms_per_step"),
                  "select_ms": base.get("roofline", {}).get("select_avg_ms")},
           "modes": {}}
    for mode in args.modes.split(","):
        rows = []
        for g in worlds:
            if g == 1:
                continue
            d = run(args, g, mode)
            if "error" in d:
                rows.append({"g": g, "error": d["error"]})
                continue
            em = d["emulated"]
            rows.append({"g": g, "local_batch": d["config"]["local_batch"],
                         "rank_ms_per_step": em["rank_ms_per_step"],
                         "comm_ms_model": em["comm_ms_model"],
                         "projected_ms_per_step": em["projected_ms_per_step"],
                         "projected_value": em["projected_value"],
                         "eff": round(em["projected_value"] / (g * v1), 4) if v1 else None,
                         "select_ms": d["roofline"]["select_avg_ms"],
                         "attend_iso_ms": d["roofline"]["avg_launch_ms"],
                         "comm_model": em["comm_model"]})
            print(mode, rows[-1], flush=True)
        out["modes"][mode] = rows
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
