"""Async vs Jacobi sweep counts per run (max over convergences) for a config:
how close the async schedule's count comes to the reference's Jacobi count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_14047_b200 as D  # noqa: E402

for cfg in sys.argv[1:] or ["c3"]:
    gen, a, m, wspec, r, k, desc = bench.CONFIGS[cfg]
    g = D.generate(gen, a, m, bench.SEED)
    ctx = D.Context(0)
    ctx.upload(g)
    out = {}
    for jac in (0, 1):
        ctx.run_json(None, k=k, r=r, weights=wspec, seed=bench.SEED, timings=False, jacobi=jac,
                     resident=True)
        st = ctx.stats()
        out[jac] = (st["max_sweeps"], st["sweeps_total"], st["rerun_jacobi"], round(st["total"], 3))
    print(cfg, "async (max, total, rerun, s):", out[0], "jacobi:", out[1], flush=True)
