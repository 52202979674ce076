#!/bin/bash
# full GPU test suite (bounded)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest tests -x -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1
echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
