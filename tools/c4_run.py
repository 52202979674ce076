"""BASELINE.json config 4 (R-MAT scale 26, 1B edges, IC p=0.005, R=1024,
K=100; quoted for 8 FASST partitions on 8 GPUs) on ONE B200: the same 8
partitions held by one context (devices=8, the reference's run_json with
devices=8 gives the identical report).  Prints generation / upload / run
times and the memory the context used.  Usage: python tools/c4_run.py [devices]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

devices = int(sys.argv[1]) if len(sys.argv) > 1 else 8
gen, a, m, wspec, r, k, desc = bench.CONFIGS["c4"]
t0 = time.time()
g = D.generate(gen, a, m, bench.SEED)
tgen = time.time() - t0
print(f"generated n={g.n} m={g.m} in {tgen:.1f}s", flush=True)
ctx = D.Context(0)
t0 = time.time()
ctx.upload(g)
torch.cuda.synchronize()
tup = time.time() - t0
st = torch.cuda.ExternalStream(ctx.stream)
out = {"workload": desc, "n": g.n, "m": g.m, "devices": devices, "generate_s": tgen,
       "upload_s": tup, "runs": []}
for i in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rep = json.loads(ctx.run_json(None, k=k, r=r, devices=devices, weights=wspec, seed=bench.SEED,
                                  timings=True, resident=True))
    e1.record(st)
    e1.synchronize()
    s = ctx.stats()
    out["runs"].append({"seconds": e0.elapsed_time(e1) / 1e3, "timings": rep["timings"],
                        "rebuilds": rep["rebuilds"], "seeds_head": rep["seeds"][:5],
                        "score": rep["score_trajectory"][-1],
                        "items_fwd": s["items_fwd"], "sketch_edge_updates": s["sketch_edge_updates"]})
    print(json.dumps(out["runs"][-1]), flush=True)
free, total = torch.cuda.mem_get_info()
out["device_mem_used_gb"] = (total - free) / 1e9
print(json.dumps(out))
