"""Per-config DRAM traffic of the attend kernel -> profiles/traffic_{config}.json
(the `roofline.traffic` bench.py reports).

Input: one ncu CSV per config (comma-separated, in the order of --configs),
each from

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:attend_kernel -c 20 --csv --log-file t_qwen7b.csv \\
        python bench.py --config qwen7b --quick --steps 1 --warmup 3 --no-cpu-baseline
    python tools/traffic.py --csv t_qwen7b.csv,t_qwen14b.csv --configs qwen7b,qwen14b

Each launch is replayed with caches flushed (ncu's default), so the bytes are
a cold launch's.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--csv", required=True)
    ap.add_argument("--configs", required=True)
    ap.add_argument("--source", default="")
    args = ap.parse_args()
    import bench
    from paper_2508_02751_b200 import bytes_model
    configs = args.configs.split(",")
    csvs = args.csv.split(",")
    if len(csvs) != len(configs):
        raise SystemExit("one CSV per config")
    per = {}
    pids = []
    for fi, path in enumerate(csvs):
        hdr = None
        for r in csv.reader(open(path)):
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                x = dict(zip(hdr, r))
                d = per.setdefault((fi, x["ID"]), {"pid": fi})
                d[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
                d["unit_" + x["Metric Name"]] = x["Metric Unit"]
        pids.append(fi)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for pid, cname in zip(pids, configs):
        ls = [d for d in per.values() if d["pid"] == pid]
        rd = [d["dram__bytes_read.sum"] * scale[d["unit_dram__bytes_read.sum"]] for d in ls]
        wr = [d["dram__bytes_write.sum"] * scale[d["unit_dram__bytes_write.sum"]] for d in ls]
        cfg = bench.workload(argparse.Namespace(config=cname, tau=None, seq_len=None))
        K, R, M = cfg.budget
        seq = [cfg.seq_len] * cfg.batch
        alg = bytes_model.step_bytes_coherent(cfg, seq, [(K, R, M)] * cfg.batch, cfg.llm.layers)["attend_per_layer"]
        out = {
            "config": cname,
            "budget": list(cfg.budget),
            "kernel": "attend_kernel",
            "launches_profiled": len(ls),
            "attend_dram_bytes_per_launch": int(sum(rd) / len(rd) + sum(wr) / len(wr)),
            "dram_read_per_launch": int(sum(rd) / len(rd)),
            "dram_write_per_launch": int(sum(wr) / len(wr)),
            "algorithmic_bytes_per_launch": int(alg),
            "traffic_over_algorithmic": round((sum(rd) / len(rd) + sum(wr) / len(wr)) / alg, 4),
            "source": args.source or f"ncu (cache flushed per replay) {os.path.basename(csvs[pid])}",
        }
        with open(os.path.join(ROOT, "profiles", f"traffic_{cname}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))


if __name__ == "__main__":
    main()
