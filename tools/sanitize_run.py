"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck): single partition, multi-partition, Jacobi + count modes, stage
API, FASST analytics and the MC oracle, each checked against the oracle.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

g = D.generate("rmat", 11, 12000, 3)
cg = O.CSR(g.offsets, g.adj, np.array(g.orig_ids, np.uint64))
ctx = D.Context(0)
for devices, r, w, extra in ((1, 128, "const:0.1", {}), (4, 256, "wc", {}), (1, 64, "const:0.2", {"jacobi": 1}),
                             (1, 96, "const:0.1", {"jacobi": 1, "count": 1})):
    got = json.loads(ctx.run_json(g, k=6, r=r, devices=devices, weights=w, seed=5, timings=False, **extra))
    want = O.run(cg, k=6, r=r, devices=devices, weights=w, seed=5)
    assert all(got[k] == v for k, v in want.items()), (devices, r, w, extra)
    print("run ok", devices, r, w, extra, flush=True)
ctx.prepare(g, r=128, devices=2, weights="const:0.1", seed=3)
ctx.fill(1)
ctx.simulate(1)
ctx.scores(1)
ctx.commit_cascade(1, 5)
print("stage ok", flush=True)
st = ctx.fasst_stats(g, r=256, devices=4, mode="fasst", weights="wc", seed=2)
assert st == O.fasst_stats(cg, 256, 4, "fasst", "wc", 2)
print("fasst_stats ok", flush=True)
m1 = ctx.influence(g, [0, 3], trials=40, seed=1, weights="const:0.1")
assert m1 == D.influence(g, [0, 3], trials=40, seed=1, weights="const:0.1")
print("influence ok", flush=True)
print("SANITIZE RUN DONE")
