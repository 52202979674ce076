"""Stage timings on a bench config (CUDA events on the context stream):
fill, simulate (one convergence), commit+cascade of the first seeds.
Usage: python tools/stage_bench.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
st = torch.cuda.ExternalStream(ctx.stream)


def timed(f, reps=3):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f()
        e1.record(st)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return " ".join(f"{x:.3f}" for x in out)


print("fill ms", timed(lambda: ctx.fill(0)))
print("simulate ms", timed(lambda: (ctx.fill(0), ctx.simulate(0)), reps=2))
print("scores(D2H incl) ms", timed(lambda: ctx.scores(0), reps=2))
del ctx, g
