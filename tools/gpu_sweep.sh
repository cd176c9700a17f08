#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --lengths 27,101,121,151,171,201,223,255,257,301,401,449,511,1023 --walk-factors 8 --seconds 1.0 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/sweep.py --lengths 301,449 --walk-factors 1,2,4,16,32 --seconds 1.0 > gpurun_out/sweep_wf.jsonl 2>> gpurun_out/sweep.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast and (large or oracle)" > gpurun_out/pytest_large.log 2>&1
echo done
