#!/bin/bash
# Round-end evidence pass: everything in gpu_full.sh, then the L=93 exhaustive scan (D=47, the scan's limit).
set -x
bash tools/gpu_full.sh
timeout 1800 python tools/exhaustive_bench.py --lengths 93 --cpu-length 0 > gpurun_out/exh_bench_93.jsonl 2> gpurun_out/exh_bench_93.err
echo done
