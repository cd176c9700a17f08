#!/bin/bash
# Config 3: lambda calibration campaigns + time-to-known-best at L=171.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python tools/time_to_target.py --lengths 71,75,79,83,101,121 --reps 100 > gpurun_out/ttt_campaign.jsonl 2> gpurun_out/ttt_campaign.err
timeout 1300 python tools/time_to_target.py --direct 171 --max-runtime 1200 > gpurun_out/ttt_direct171.jsonl 2> gpurun_out/ttt_direct171.err
echo done
