#!/bin/bash
# A/B of two package builds (exp/<name>pkg vs the working tree) on one config
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in ${CFGS:-c3ic}; do
for rep in 1 2; do
  for pkg in ${PKGS:-exp/r1pkg .}; do
    DFS_PKG=$pkg timeout 300 python tools/profile_run.py $cfg 3 2>gpurun_out/ab_err.txt | tail -1 > gpurun_out/ph.txt
    python - $pkg $cfg <<'PY'
import ast, sys
d = ast.literal_eval(open("gpurun_out/ph.txt").read())
print(sys.argv[2], sys.argv[1], {k: round(d[k] * 1e3, 2) for k in ("build", "fill", "simulate", "select", "cascade", "total")}, "krun", round(d["run_kernel"] * 1e3, 2), "density", round(d.get("item_density", 0), 3), "sweeps", d["sweeps_total"])
PY
  done
done
done
