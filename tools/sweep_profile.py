"""Per-sweep cost of the simulate kernel: time simulate(cap=c) from a fresh
fill for c = 1..; differences are per-sweep costs.  Also cascade per seed."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
prev = 0.0
for cap in range(1, 40):
    ctx.fill(0)
    t0 = time.perf_counter()
    try:
        sw = ctx.simulate(0, cap=cap)
        done = True
    except RuntimeError:
        sw, done = cap, False
    dt = time.perf_counter() - t0
    c = ctx.counters(0)
    print(f"cap {cap:2d} sweeps {sw:2d} time {dt*1e3:8.3f} ms  delta {1e3*(dt-prev):8.3f}  items {c['items']}")
    prev = dt
    if done:
        break
rep = ctx.run_json(None, k=k, r=r, weights=wspec, seed=bench.SEED, timings=False, resident=True)
import json  # noqa: E402
seeds = json.loads(rep)["seeds_dense"]
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
ctx.fill(0)
ctx.simulate(0)
for i, s in enumerate(seeds[:12]):
    t0 = time.perf_counter()
    v = ctx.commit_cascade(0, s)
    dt = time.perf_counter() - t0
    print(f"cascade {i:2d} seed {s:7d} visited {v:10d} {dt*1e6:9.1f} us")
