"""BASELINE.json config 5: register-count / simulation sweep on the scale-23
R-MAT (100M edges, IC p=0.01, K=50).  Registers = simulations in the
reference (one int8 register per (vertex, simulation)); the per-GPU register
slice is J = R / devices, so "8-64 sketch registers" is swept as R = 64..512
over 8 FASST partitions (J = 8..64; J < 32 is the reference's degraded plan).
The estimate is bit-identical to the CPU reference by construction (tested),
so the error reported is the estimate vs the Monte-Carlo influence of the
selected seeds (GPU oracle, bit-identical to the reference's influence()).
Usage: python tools/c5_sweep.py [mc_trials]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
gen, a, m, wspec, r0, k, desc = bench.CONFIGS["c3ic"]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.upload(g)
st = torch.cuda.ExternalStream(ctx.stream)
rows = []
for devices, rs in ((1, (64, 128, 256, 512, 1024, 2048, 4096)), (8, (64, 128, 256, 512))):
    for r in rs:
        ts = []
        for i in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rep = json.loads(ctx.run_json(None, k=k, r=r, devices=devices, weights=wspec,
                                          seed=bench.SEED, timings=False, resident=True))
            e1.record(st)
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) / 1e3)
        s = ctx.stats()
        est = rep["score_trajectory"][-1]
        mc, se = ctx.influence(None, rep["seeds_dense"], trials=trials, seed=1, weights=wspec,
                               resident=True)
        row = {"r": r, "devices": devices, "J": r // devices, "degraded": rep["degraded_plan"],
               "seconds": round(statistics.mean(ts), 5), "rebuilds": rep["rebuilds"],
               "simulate_s": round(s["simulate"], 5), "sketch_edge_updates": s["sketch_edge_updates"],
               "updates_per_s": s["sketch_edge_updates"] / max(s["simulate"], 1e-12),
               "estimate": est, "mc_influence": mc, "mc_std_error": se, "mc_trials": trials,
               "rel_error_vs_mc": (est - mc) / mc if mc else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
out = {"workload": desc + " (config 5 sweep)", "n": g.n, "m": g.m, "rows": rows}
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                       "c5_sweep.json"), "w") as f:
    json.dump(out, f, indent=1)
