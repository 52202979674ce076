import os, sys, time, json
sys.path.insert(0, "/root/repo")
import torch, bench
import paper_2410_14047_b200 as D
g = D.generate("rmat", 20, 16_000_000, 7)
ctx = D.Context(0); ctx.upload(g)
st = torch.cuda.ExternalStream(ctx.stream)
flush = torch.empty(256*1024*1024//4, dtype=torch.int32, device="cuda")
for i in range(8):
    flush.add_(1); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    rep = ctx.run_json(None, k=50, r=256, weights="const:0.01", seed=7, timings=True, resident=True)
    t1 = time.perf_counter(); e1.record(st); e1.synchronize(); t2 = time.perf_counter()
    tm = json.loads(rep)["timings"]
    print(f"event {e0.elapsed_time(e1):7.3f} ms  host call {1e3*(t1-t0):7.3f}  total {1e3*tm['total']:7.3f} build {1e3*tm['build']:6.3f}")
