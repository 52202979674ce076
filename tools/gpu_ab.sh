#!/bin/bash
# quick A/B: parity subset + phase times per config (3 runs each, last printed)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_quick.log 2>&1
echo pytest_rc=$? $(tail -1 gpurun_out/pytest_quick.log)
for cfg in ${CFGS:-c2 c3ic}; do
  timeout 300 python tools/profile_run.py $cfg 3 2>&1 | tail -1 > gpurun_out/phases_$cfg.txt
  python - $cfg <<'PY'
import ast, sys
c = sys.argv[1]
d = ast.literal_eval(open(f"gpurun_out/phases_{c}.txt").read())
print(c, {k: round(d[k] * 1e3, 2) for k in ("build", "fill", "simulate", "select", "cascade", "total")},
      "sweeps", d["sweeps_total"], "krun_ms", round(d["run_kernel"] * 1e3, 2))
PY
done
