#!/bin/bash
# Kernel iteration: fast-evaluator parity subset, bench, one ncu --set full capture.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast" > gpurun_out/pytest_fast.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err
timeout 600 python tools/sweep.py --lengths 101,201,301,449 --walk-factors 8 --seconds 1.0 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/prof_fast -f \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 65536 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
fi
echo done
