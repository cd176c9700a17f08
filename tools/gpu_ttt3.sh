#!/bin/bash
# Config 3: long time-to-known-best runs at L=193 and L=199 (published targets).
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2500 python tools/time_to_target.py --direct 193 --seed 7 --max-runtime 2400 > gpurun_out/ttt_193.jsonl 2> gpurun_out/ttt_193.err
echo done
