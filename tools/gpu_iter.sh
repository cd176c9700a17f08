#!/bin/bash
# quick iteration: fast-variant parity subset + bench + one ncu capture
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast and (goldens or oracle)" > gpurun_out/pytest_fast.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --variant fast --no-cpu-baseline --no-e2e > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/prof_fast -f \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 32768 --variant fast --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
fi
echo done
