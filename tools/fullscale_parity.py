"""Full-scale parity: the same configuration through our GPU path and through
the UNMODIFIED reference (oracle/_ref, its own pybind run_json) on this host,
reports compared byte for byte (timings excluded).  Both sides use
devices = D sample-space partitions (ours: D partitions in one context on one
GPU; the reference: D worker threads), so the seed sets must be identical.
Usage: python tools/fullscale_parity.py [config] [devices]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3ic"
devices = int(sys.argv[2]) if len(sys.argv) > 2 else 16
gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
g = D.generate(gen, a, m, bench.SEED)
ctx = D.Context(0)
t0 = time.perf_counter()
ours = ctx.run_json(g, k=k, r=r, devices=devices, weights=wspec, seed=bench.SEED, timings=False)
t_ours = time.perf_counter() - t0
ref, _ = O.load_reference()
if ref is None:
    sys.exit("reference build (oracle/_ref) missing")
path = f"/tmp/fullscale_{os.getpid()}.bin"
D.save_cache(g, path)
rg = ref.load_graph(path)
os.unlink(path)
t0 = time.perf_counter()
theirs = ref.run_json(rg, k=k, r=r, devices=devices, mode="fasst", weights=wspec, rebuild_eps=0.01,
                      seed=bench.SEED, timings=False)
t_ref = time.perf_counter() - t0
a_, b_ = json.loads(ours), json.loads(theirs)
out = {"workload": desc, "n": g.n, "m": g.m, "devices": devices,
       "byte_identical_report": ours == theirs,
       "seeds_equal": a_["seeds"] == b_["seeds"],
       "trajectory_equal": a_["score_trajectory"] == b_["score_trajectory"],
       "rebuild_rounds_equal": a_["rebuild_rounds"] == b_["rebuild_rounds"],
       "seeds_head": a_["seeds"][:10], "final_score": a_["score_trajectory"][-1],
       "ours_s_incl_upload": round(t_ours, 3), "reference_s": round(t_ref, 3),
       "reference_threads": devices}
print(json.dumps(out))
