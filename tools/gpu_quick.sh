#!/bin/bash
# quick check: parity subset + launch lists of C2 and the north star
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -rs > gpurun_out/pytest_quick.log 2>&1
echo pytest_rc=$?
for cfg in ${CFGS:-c2 c3ic}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$cfg.csv python tools/profile_run.py $cfg 2 > gpurun_out/prof_$cfg.log 2>&1
echo launches_rc=$?
done
