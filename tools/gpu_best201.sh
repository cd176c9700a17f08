#!/bin/bash
# Best energy found at L=201 (the headline length; no published target) in ~50 min on one B200.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 3200 python -m paper_2210_15962_b200 solve --length 201 --walkers 1048576 --seed 2026 --max-runtime 3000 > gpurun_out/best201.json 2> gpurun_out/best201.err
echo done
