#!/bin/bash
# Full ncu capture of the persistent greedy-loop kernel k_run at a bench config
# (default: the north star c3ic).  Usage: bash tools/gpu_ncu_c3ic.sh [config] [tag]
cfg=${1:-c3ic}; tag=${2:-$cfg}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'^k_run$' -c 1 \
   -o gpurun_out/krun_$tag -f python tools/profile_run.py $cfg 1 > gpurun_out/krun_$tag.log 2>&1
echo ncu_rc=$?
