"""Per-level device trace of one resident run (DFS_DBG=4 must be set before
the process starts): sim/cas level records with frontier sizes and clock
deltas, round/rescored/argmax/chosen markers.  Usage:
DFS_DBG=4 python tools/trace_run.py [cfg] 2> trace.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
if os.environ.get("DFS_PKG"):  # another build of the package (A/B)
    sys.path.insert(0, os.environ["DFS_PKG"])
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.upload(g)
for i in range(2):
    print(f"== run {i}", file=sys.stderr, flush=True)
    ctx.run_json(None, k=k, r=r, weights=wspec, seed=bench.SEED, timings=True, resident=True)
