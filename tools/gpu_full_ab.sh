#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo gpu rc=$? $(tail -1 gpurun_out/pytest_gpu.log)
PKGS="exp/headpkg ." CFGS="c2 c3" bash tools/gpu_ab_pkg.sh
