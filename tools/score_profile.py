"""Full rescore (k_score over every row) of the north-star partition after
the first convergence, timed with CUDA events; run under ncu with
-k regex:k_score -c 1 for the kernel profile.  Usage: python tools/score_profile.py [cfg]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3ic"
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, k=k, r=r, weights=wspec, seed=bench.SEED)
ctx.fill(0)
ctx.simulate(0)
st = torch.cuda.ExternalStream(ctx.stream)
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.scores(0)
    e1.record(st)
    e1.synchronize()
    print("scores ms (incl. D2H of n doubles)", e0.elapsed_time(e1))
