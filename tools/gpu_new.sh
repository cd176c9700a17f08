#!/bin/bash
# New-component pass: exhaustive scan + campaign tests, exhaustive throughput.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_campaign.py -m gpu -x -q > gpurun_out/pytest_new.log 2>&1
timeout 600 python tools/exhaustive_bench.py --lengths 45,55,61,65,71 --cpu-length 41 > gpurun_out/exh_bench.jsonl 2> gpurun_out/exh_bench.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo done
