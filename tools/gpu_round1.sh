#!/bin/bash
# First GPU pass: smoke, microbench, gpu tests, short bench, launch list.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 tools/microbench > gpurun_out/microbench.json 2> gpurun_out/microbench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --cpu-seconds 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --walkers-per-gpu 65536 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
echo done
