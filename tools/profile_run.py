"""One resident IM run of a bench config (for ncu launch lists / captures).
Usage: python tools/profile_run.py [config] [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (puts the repo root first on sys.path)
if os.environ.get("DFS_PKG"):  # A/B against another build of the package
    sys.path.insert(0, os.environ["DFS_PKG"])
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.upload(g)
for _ in range(runs):
    rep = ctx.run_json(None, k=k, r=r, devices=int(os.environ.get("DEVICES", "1")), weights=wspec,
                       seed=bench.SEED, timings=True, resident=True)
print(rep)
print(ctx.stats())
