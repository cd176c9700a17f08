#!/bin/bash
# lambda(L) calibration on exact targets: campaigns of 100 concurrent repetitions at L=71..87,
# each target the exact optimum from the device exhaustive scan; exhaustive scans up to L=91;
# then the A/B of pending variants.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 1800 python tools/time_to_target.py --lengths 71,73,75,77,79,81,83,85,87 --reps 100 --exhaustive-max-d 44 > gpurun_out/calib_exact.jsonl 2> gpurun_out/calib_exact.err
timeout 1500 python tools/exhaustive_bench.py --lengths 89,91 --cpu-length 0 > gpurun_out/exh_bench_89_91.jsonl 2> gpurun_out/exh_bench_89_91.err
bash tools/gpu_ab.sh
echo done
