#!/bin/bash
# A/B of a DFS_DBG knob: phase times per config, alternating A and B runs
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in ${CFGS:-c2 c3ic}; do
  for rep in 1 2; do
    for v in ${VARIANTS:-0 16}; do
      DFS_DBG=$v timeout 300 python tools/profile_run.py $cfg 3 2>&1 | tail -1 > gpurun_out/ph.txt
      python - $cfg $v <<'PY'
import ast, sys
c, v = sys.argv[1], sys.argv[2]
d = ast.literal_eval(open("gpurun_out/ph.txt").read())
print(c, "dbg", v, {k: round(d[k] * 1e3, 2) for k in ("build", "fill", "simulate", "select", "cascade", "total")}, "krun", round(d["run_kernel"] * 1e3, 2))
PY
    done
  done
done
