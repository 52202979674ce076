"""Monte-Carlo influence (oracle.cpp:30-79) on the GPU vs the reference's
CPU influence() on the same graph / seeds / trials (seconds per trial).
Usage: python tools/mc_bench.py [config] [gpu_trials] [cpu_trials]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gt = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
ct = int(sys.argv[3]) if len(sys.argv) > 3 else 16
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
rep = json.loads(ctx.run_json(g, k=k, r=r, weights=wspec, seed=bench.SEED, timings=False))
seeds = rep["seeds_dense"]
ctx.influence(g, seeds, trials=64, seed=1, weights=wspec)  # warm-up (upload, allocations)
t0 = time.perf_counter()
mean, se = ctx.influence(g, seeds, trials=gt, seed=1, weights=wspec, resident=True)
tg = time.perf_counter() - t0
out = {"workload": desc, "seeds": len(seeds), "gpu_trials": gt, "gpu_s": tg,
       "gpu_s_per_trial": tg / gt, "gpu_mean": mean, "gpu_std_error": se,
       "sketch_estimate": rep["score_trajectory"][-1]}
ref, _ = O.load_reference()
if ref is not None and ct:
    path = f"/tmp/mc_{os.getpid()}.bin"
    D.save_cache(g, path)
    rg = ref.load_graph(path)
    os.unlink(path)
    t0 = time.perf_counter()
    rm, rs = ref.influence(rg, seeds, trials=ct, seed=1, weights=wspec)
    tc = time.perf_counter() - t0
    gm, gs = ctx.influence(g, seeds, trials=ct, seed=1, weights=wspec, resident=True)
    out.update({"cpu_trials": ct, "cpu_s": tc, "cpu_s_per_trial": tc / ct, "cpu_threads": 1,
                "bit_identical_at_cpu_trials": (gm, gs) == (rm, rs),
                "speedup_per_trial": (tc / ct) / (tg / gt)})
print(json.dumps(out))
