#!/bin/bash
# A/B of experimental builds (libsokol_<name>.so) against libsokol.so: throughput sweep per variant, twice.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
LENS=${LENS:-101,151,201,255,301,449}
for rep in 1 2; do
for lib in paper_2210_15962_b200/libsokol*.so; do
  name=$(basename $lib .so)
  SOKOL_LIB=$PWD/$lib timeout 300 python tools/sweep.py --lengths $LENS --walk-factors 8 --seconds 1.0 > gpurun_out/var_${name}_$rep.jsonl 2> gpurun_out/var_${name}_$rep.err
done
done
echo done
