"""Simulate time vs R on one graph (does a 32-sim batch converge faster
alone than its share of a wide run?).  Usage: python tools/batch_probe.py cfg"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
gen, a, m, wspec, r0, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
st = None
for r in (32, 64, 128, 256, 1024):
    ctx.prepare(g, r=r, weights=wspec, seed=bench.SEED)
    st = torch.cuda.ExternalStream(ctx.stream)
    ts = []
    for _ in range(3):
        ctx.fill(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw = ctx.simulate(0)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    c = ctx.counters(0)
    print(f"{cfg} R={r:5d} simulate {min(ts):8.3f} ms  per-32-batch {min(ts) * 32 / r:7.3f} ms  sweeps {sw}  items {c['items']}", flush=True)
