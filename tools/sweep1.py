import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2410_14047_b200 as D
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
ts = []
for rep in range(5):
    ctx.fill(0)
    t0 = time.perf_counter()
    try:
        ctx.simulate(0, cap=1)
    except RuntimeError:
        pass
    ts.append(time.perf_counter() - t0)
print(os.environ.get("DFS_DBG", "0"), "sweep1 ms", [round(t * 1e3, 3) for t in ts])
