#!/bin/bash
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python tools/config5.py --lengths 301,449 --walk-factors 1,2,4,8,16,32 --seconds 30 > gpurun_out/config5.jsonl 2> gpurun_out/config5.err
timeout 600 python -m pytest tests/test_gpu_acceptance.py -m gpu -q -k "criterion_6" > gpurun_out/pytest_c6.log 2>&1
echo done
