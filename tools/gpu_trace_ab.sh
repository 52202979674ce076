#!/bin/bash
# per-level device traces of one config for two package builds
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for pkg in ${PKGS:-exp/r1pkg .}; do
  tag=$(echo $pkg | tr '/.' '__')
  DFS_PKG=$pkg DFS_DBG=4 timeout 300 python tools/trace_run.py ${CFG:-c3} 2> gpurun_out/trace_$tag.txt > /dev/null
  echo $pkg rc=$?
done
