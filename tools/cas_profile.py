"""One commit+cascade of C2's first seed (the giant cascade: ~70% of C2's
cascade time) as a stand-alone k_cascade launch, for ncu source profiling.
Usage: ncu -k regex:k_cascade -c 1 ... python tools/cas_profile.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

gen, a, m, wspec, r, k, desc = bench.CONFIGS["c2"]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
ctx.fill(0)
ctx.simulate(0)
st = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
ctx.commit_cascade(0, 0)
e1.record(st)
e1.synchronize()
print("cascade ms", e0.elapsed_time(e1))
