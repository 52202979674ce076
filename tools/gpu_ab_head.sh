#!/bin/bash
# parity subset + A/B of the working tree against exp/headpkg (a build of HEAD)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_parity.log 2>&1
echo parity rc=$? $(tail -1 gpurun_out/pytest_parity.log)
PKGS="exp/headpkg ." CFGS="${CFGS:-c2 c3ic}" bash tools/gpu_ab_pkg.sh
