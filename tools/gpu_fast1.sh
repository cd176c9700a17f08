#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 tools/microbench > gpurun_out/microbench.json 2> gpurun_out/microbench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast and (goldens or oracle)" > gpurun_out/pytest_fast.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --variant fast --cpu-seconds 5 --no-e2e > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/prof_fast \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 32768 --variant fast --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo done
