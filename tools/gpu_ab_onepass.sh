#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_parity.log 2>&1
echo parity rc=$? $(tail -1 gpurun_out/pytest_parity.log)
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "bench_workload or 16m or r1024" > gpurun_out/pytest_scale.log 2>&1
echo scale rc=$? $(tail -1 gpurun_out/pytest_scale.log)
PKGS="exp/basepkg ." CFGS="c2 c3ic c3" bash tools/gpu_ab_pkg.sh
