#!/bin/bash
# New-component pass: exhaustive scan + campaign + neighbourhood tests, then the full GPU suite.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_campaign.py tests/test_gpu_neighborhood.py -m gpu -q > gpurun_out/pytest_new.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo done
