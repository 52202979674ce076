#!/bin/bash
# round-end measurement set: bench lines (C2 headline with the north star, the north-star line),
# launch lists, C4 on one GPU, partition projection, k_run captures (c2, c3ic)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc=$?
timeout 600 python bench.py --config c3ic --steps 5 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/bench_c3ic.json 2> gpurun_out/bench_c3ic.err; echo c3ic rc=$?
for cfg in c2 c3ic; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$cfg.csv python tools/profile_run.py $cfg 2 > gpurun_out/prof_$cfg.log 2>&1; echo ll $cfg rc=$?
done
timeout 900 python tools/partition_projection.py c3ic 8 > gpurun_out/projection.jsonl 2>&1; echo proj rc=$?
timeout 1200 python tools/c4_run.py 8 > gpurun_out/c4.json 2>&1; echo c4 rc=$?
# k_run captures: summaries extracted on the box (full .ncu-rep files exceed the copy-back limit)
for cfg in c2 c3ic; do
  bash tools/gpu_ncu_kernel.sh '^k_run$' $cfg krun_$cfg 0
  python tools/ncu_summary.py gpurun_out/ncu_krun_$cfg.ncu-rep > gpurun_out/ncu_krun_$cfg.txt 2>&1
  python tools/ncu_lines.py gpurun_out/ncu_krun_$cfg.ncu-rep >> gpurun_out/ncu_krun_$cfg.txt 2>&1
  rm -f gpurun_out/ncu_krun_$cfg.ncu-rep
done
