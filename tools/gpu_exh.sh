#!/bin/bash
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_campaign.py -m gpu -q > gpurun_out/pytest_exh.log 2>&1
timeout 900 python tools/exhaustive_bench.py --lengths 45,55,61,65,71,75,79 --cpu-length 41 > gpurun_out/exh_bench.jsonl 2> gpurun_out/exh_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exhaustive_kernel -c 1 -o gpurun_out/prof_exh -f \
    python tools/exhaustive_bench.py --lengths 71 --cpu-length 0 > gpurun_out/ncu_exh.log 2>&1
echo done
