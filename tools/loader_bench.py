"""Host graph substrate timings: generator, DFSG0001
save, DFSG0001 load for the product (paper_2410_14047_b200) and, when the
compiled reference exists (oracle/_ref), the reference's own load_graph of the
same cache file.  Usage: python tools/loader_bench.py [config ...] > out.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

ref, _ = O.load_reference()
for cfg in sys.argv[1:] or ["c2", "c3ic"]:
    gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
    path = f"/tmp/loader_{cfg}.bin"
    t0 = time.perf_counter()
    g = D.generate(gen, a, m, bench.SEED)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    D.save_cache(g, path)
    t_save = time.perf_counter() - t0
    del g
    t0 = time.perf_counter()
    g = D.load_graph(path)
    t_load = time.perf_counter() - t0
    out = {"config": cfg, "workload": desc, "n": g.n, "m": g.m,
           "bytes": os.path.getsize(path), "threads": os.cpu_count(),
           "generate_s": round(t_gen, 3), "save_s": round(t_save, 3), "load_s": round(t_load, 3)}
    del g
    if ref is not None:
        t0 = time.perf_counter()
        rg = ref.load_graph(path)
        out["reference_load_s"] = round(time.perf_counter() - t0, 3)
        del rg
    os.remove(path)
    print(json.dumps(out), flush=True)
