#!/bin/bash
# A/B of library builds incl. the build phase: tools/ab_build.sh cfg reps lib1 lib2 ...
cfg=$1; reps=$2; shift 2
for L in "$@"; do
  for i in $(seq $reps); do
    echo -n "$L $cfg: "
    DFS_LIB=$PWD/$L/libdifuser_b200.so timeout 300 python tools/profile_run.py $cfg 2 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print({k: round(d[k]*1e3,3) for k in ('build','simulate','cascade','total')})"
  done
done
