#!/bin/bash
# Config 3: more seeds for the time-to-known-best distribution at L=185 and L=193.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1700 python tools/time_to_target.py --direct 185 --seed 2 --direct-seeds 5 --max-runtime 300 > gpurun_out/ttt_185x5.jsonl 2> gpurun_out/ttt_185x5.err
timeout 2000 python tools/time_to_target.py --direct 193 --seed 8 --direct-seeds 2 --max-runtime 900 > gpurun_out/ttt_193x2.jsonl 2> gpurun_out/ttt_193x2.err
echo done
