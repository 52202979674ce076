for cfg in c2 c3ic; do for cp in 2 4 8 16 64 100000; do
  echo -n "CAS_PULL=$cp $cfg: "
  DFS_CAS_PULL=$cp timeout 300 python tools/profile_run.py $cfg 2 2>&1 | tail -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print({k: round(d[k]*1e3,3) for k in ('simulate','cascade','select','total')})"
done; done
