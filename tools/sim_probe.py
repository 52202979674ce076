"""One fill + simulate of a bench config through the stage API (for ncu
captures of k_simulate and quick timing).  Usage: python tools/sim_probe.py [cfg] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
for _ in range(reps):
    ctx.fill(0)
    ctx.simulate(0)  # warm
    ctx.fill(0)
    t0 = time.perf_counter()
    sw = ctx.simulate(0)
    dt = time.perf_counter() - t0
    print(f"{cfg} slab={os.environ.get('DFS_SLAB', 'auto')} simulate {dt * 1e3:.3f} ms sweeps {sw} "
          f"counters {ctx.counters(0)}", flush=True)
