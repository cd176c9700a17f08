#!/bin/bash
# Config 3: long time-to-known-best runs at L=199 and L=197 (published targets).
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2500 python tools/time_to_target.py --direct 199 --seed 7 --max-runtime 2400 > gpurun_out/ttt_199.jsonl 2> gpurun_out/ttt_199.err
timeout 2500 python tools/time_to_target.py --direct 197 --seed 7 --max-runtime 2400 > gpurun_out/ttt_197.jsonl 2> gpurun_out/ttt_197.err
echo done
