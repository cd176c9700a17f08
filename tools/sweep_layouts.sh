#!/bin/bash
# Throughput per (evaluator variant, visited layout): SK_SWEEP_VARIANT / SK_SWEEP_LAYOUT read by tools/sweep.py
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
LENS=${LENS:-101,151,201,255,301,449}
for v in fast; do for lay in 0 1 2 3; do
  SK_SWEEP_LAYOUT=$lay timeout 300 python tools/sweep.py --variant $v --lengths $LENS --walk-factors 8 --seconds 1.0 > gpurun_out/lay_${v}_$lay.jsonl 2> gpurun_out/lay_${v}_$lay.err
done; done
echo done
