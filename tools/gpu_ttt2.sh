#!/bin/bash
# Config 3: time-to-known-best at the published lengths (direct solves, several seeds).
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python tools/time_to_target.py --direct 171 --direct-seeds 5 --max-runtime 200 > gpurun_out/ttt_direct171x5.jsonl 2> gpurun_out/ttt2.err
timeout 2400 python tools/time_to_target.py --direct 185,193,197,199 --max-runtime 540 > gpurun_out/ttt_direct_more.jsonl 2>> gpurun_out/ttt2.err
echo done
