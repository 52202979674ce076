#!/bin/bash
# peer/scale tests + bench lines (default headline and the north star)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -m gpu -rs > gpurun_out/pytest_peer.log 2>&1
echo peer_rc=$? $(tail -1 gpurun_out/pytest_peer.log)
timeout 600 python bench.py --config c3ic --steps 5 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/bench_c3ic.json 2> gpurun_out/bench_c3ic.err
echo c3ic_rc=$?
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo c2_rc=$?
