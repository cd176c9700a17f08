#!/bin/bash
# A/B: fast-evaluator parity with the candidate build, then throughput sweeps of every libsokol*.so.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast" > gpurun_out/pytest_fast.log 2>&1
bash tools/gpu_variants.sh
echo done
