#!/bin/bash
# A/B of experimental builds (libsokol_<name>.so) against libsokol.so: throughput sweep per variant.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for lib in paper_2210_15962_b200/libsokol*.so; do
  name=$(basename $lib .so)
  SOKOL_LIB=$PWD/$lib timeout 300 python tools/sweep.py --lengths 101,201,255,449 --walk-factors 8 --seconds 1.0 > gpurun_out/var_$name.jsonl 2> gpurun_out/var_$name.err
done
echo done
