#!/bin/bash
# Config 3: a second, longer L=197 attempt (published E=2162).
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 3800 python tools/time_to_target.py --direct 197 --seed 8 --max-runtime 3600 > gpurun_out/ttt_197b.jsonl 2> gpurun_out/ttt_197b.err
echo done
