#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
DEVICES=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_c3ic_mu8.csv python tools/profile_run.py c3ic 1 > gpurun_out/prof_c3ic_mu8.log 2>&1
echo rc=$?
DFS_PREP_TRACE=1 DEVICES=8 timeout 600 python tools/profile_run.py c3ic 2 > gpurun_out/prep_c3ic_mu8.log 2>&1
echo rc=$?
timeout 600 python tools/loader_bench.py c2 c3ic > gpurun_out/loader.json 2>&1
echo rc=$?
