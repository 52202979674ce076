#!/bin/bash
# parity subset + per-config phase times / sweep counts (+ c3ic trace)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_quick.log 2>&1
echo pytest_rc=$?
for cfg in ${CFGS:-c2 c3ic c3}; do
  timeout 300 python tools/profile_run.py $cfg 3 2>&1 | tail -1 > gpurun_out/phases_$cfg.txt
done
DFS_DBG=4 timeout 300 python tools/trace_run.py c3ic 2> gpurun_out/trace_c3ic.txt > /dev/null
echo done
