"""BASELINE.json config 5: register-count / simulation sweep on the scale-23
R-MAT (100M edges, IC p=0.01, K=50), one GPU.

Registers = simulations in the reference (one int8 register per (vertex,
simulation)); the per-partition register slice is J = R / devices, so the
"8-64 sketch registers" range is swept as R = 64..512 over 8 FASST partitions
(J = 8..64; J < 32 is the reference's degraded plan) next to R = 64..4096 at
devices = 1 and 16.  Per row:
  * seconds (resident, CUDA events), rebuilds, sketch-edge updates/s;
  * roofline: SURVEY §8(d) algorithmic bytes of the whole loop (instrumented
    Jacobi replay, the numerator tests/test_gpu_scale.py pins to the reference's
    own stages) / the k_run launch time, and the simulate phase's fraction;
  * report parity against the reference's report of the same (R, devices)
    (tests/golden/bench_reports.json) where recorded;
  * the estimate vs the Monte-Carlo influence of the selected seeds (GPU
    oracle, bit-identical to the reference's influence()).
Usage: python tools/c5_sweep.py [mc_trials] [out]"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "c5_sweep.json")
gen, a, m, wspec, r0, k, desc = bench.CONFIGS["c3ic"]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.upload(g)
st = torch.cuda.ExternalStream(ctx.stream)
peak, peak_kind = bench.measured_peak()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
rows = []
plan = [(1, (64, 128, 256, 512, 1024, 2048, 4096)), (8, (64, 128, 256, 512)),
        (16, (64, 128, 256, 512, 1024, 2048, 4096))]
for devices, rs in plan:
    for r in rs:
        cfg = f"c5_r{r}"
        ts, krun = [], []
        for i in range(3):
            flush.add_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rep_s = ctx.run_json(None, k=k, r=r, devices=devices, weights=wspec, seed=bench.SEED,
                                 timings=False, resident=True)
            e1.record(st)
            e1.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) / 1e3)
                krun.append(ctx.stats()["run_kernel"])
        s = ctx.stats()
        rep = json.loads(rep_s)
        alg = bench.algorithmic_bytes(D, ctx, g, cfg, devices)
        kr = statistics.mean(krun)
        per_conv = s["sim_active"] / max(s["sim_launches"], 1)
        est = rep["score_trajectory"][-1]
        mc, se = ctx.influence(None, rep["seeds_dense"], trials=trials, seed=1, weights=wspec,
                               resident=True)
        row = {"r": r, "devices": devices, "J": r // devices, "degraded": rep["degraded_plan"],
               "seconds": round(statistics.mean(ts), 5), "rebuilds": rep["rebuilds"],
               "report_parity": bench.parity_of(cfg, devices, rep_s),
               "simulate_s": round(s["simulate"], 5),
               "sketch_edge_updates_per_s": s["sketch_edge_updates"] / max(s["sim_active"], 1e-12),
               "roofline": {"kernel": "k_run", "alg_bytes": alg["run_bytes"],
                            "launch_ms": round(kr * 1e3, 3),
                            "achieved_gbs": round(alg["run_bytes"] / kr / 1e9, 1),
                            "frac": round(alg["run_bytes"] / kr / 1e9 / peak, 4),
                            "frac_performed": round(alg["run_bytes_performed"] / kr / 1e9 / peak, 4),
                            "simulate_frac": round(alg["bytes_per_launch"] / per_conv / 1e9 / peak
                                                   if per_conv > 0 else 0.0, 4),
                            "peak_gbs": peak, "peak_source": peak_kind},
               "estimate": est, "mc_influence": mc, "mc_std_error": se, "mc_trials": trials,
               "rel_error_vs_mc": (est - mc) / mc if mc else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
        torch.cuda.empty_cache()
out = {"workload": desc + " (config 5 sweep)", "n": g.n, "m": g.m, "l2": "flushed between runs",
       "rows": rows}
with open(out_path, "w") as f:
    json.dump(out, f, indent=1)
