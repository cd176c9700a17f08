#!/bin/bash
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exhaustive_kernel -s 1 -c 1 -o gpurun_out/prof_exh -f \
    python tools/exhaustive_bench.py --lengths 71 --cpu-length 0 > gpurun_out/ncu_exh.log 2>&1
timeout 900 python tools/exhaustive_bench.py --lengths 83,87 --cpu-length 0 > gpurun_out/exh_bench_big.jsonl 2> gpurun_out/exh_bench_big.err
echo done
