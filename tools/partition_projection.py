"""Projection aid for multi-GPU scaling (NOT a multi-GPU measurement): runs a
configuration with devices = mu FASST partitions held by ONE context on one
GPU (the partitions' fill / simulate / cascade phases run one after another),
and reports the per-phase times.  Each of mu GPUs would own one partition, so
the partition-parallel phases divide by ~mu while the per-round exchange is
extra.  Usage: python tools/partition_projection.py cfg mu"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3ic"
mu = int(sys.argv[2]) if len(sys.argv) > 2 else 8
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.upload(g)
for devices in (1, mu):
    for i in range(2):
        rep = json.loads(ctx.run_json(None, k=k, r=r, devices=devices, weights=wspec, seed=bench.SEED,
                                      timings=True, resident=True))
    t = rep["timings"]
    print(json.dumps({"workload": desc, "devices": devices, "one_gpu_s": round(t["total"], 4),
                      "phases_ms": {x: round(1e3 * t[x], 2) for x in ("build", "fill", "simulate",
                                                                       "select", "cascade")},
                      "rebuilds": rep["rebuilds"]}))
