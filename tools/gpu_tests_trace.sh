#!/bin/bash
# GPU test suite + a per-level device trace of the north star.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo pytest_rc=$?
DFS_DBG=4 timeout 300 python tools/trace_run.py c3ic 2> gpurun_out/trace_c3ic.txt > /dev/null
echo trace_rc=$?
