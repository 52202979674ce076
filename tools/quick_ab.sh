#!/bin/bash
# Phase times (ms) of the default build on a few configs: tools/quick_ab.sh cfg...
for cfg in "$@"; do
  echo -n "$cfg: "
  timeout 300 python tools/profile_run.py $cfg 2 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print({k: round(d[k]*1e3,3) for k in ('build','fill','simulate','cascade','select','total')})"
done
