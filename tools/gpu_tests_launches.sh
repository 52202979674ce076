#!/bin/bash
# GPU test suite + launch lists of C2 and the north star.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo pytest_rc=$?
for cfg in c2 c3ic; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$cfg.csv python tools/profile_run.py $cfg 2 > gpurun_out/prof_$cfg.log 2>&1
echo launches_rc=$?
done
