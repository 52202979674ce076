#!/bin/bash
# Full ncu capture of one launch of kernel $1 during tools/profile_run.py $2 (env passed through)
# Usage: [DEVICES=8] bash tools/gpu_ncu_kernel.sh k_items_sparse c3ic tag [skip]
k=$1; cfg=${2:-c3ic}; tag=${3:-$1}; skip=${4:-0}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $skip -c 1 \
   -o gpurun_out/ncu_$tag -f python tools/profile_run.py $cfg 1 > gpurun_out/ncu_$tag.log 2>&1
echo ncu_rc=$?
