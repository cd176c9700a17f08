#!/bin/bash
# BASELINE configs 3 and 5 with the round-2 evaluator: time to the published
# best-known energies at L=171 and L=185, and the walk-factor sweep at L=301/449.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-cfg}
timeout 900 python tools/config5.py --lengths 301,449 --walk-factors 1,2,4,8,16,32 --seconds 20 > gpurun_out/${T}_config5.jsonl 2> gpurun_out/${T}_config5.err; echo "config5 rc=$?"
timeout 900 python tools/time_to_target.py --direct 171 --seed 1 --direct-seeds 5 --max-runtime 150 > gpurun_out/${T}_ttt_171.jsonl 2> gpurun_out/${T}_ttt_171.err; echo "ttt171 rc=$?"
timeout 1500 python tools/time_to_target.py --direct 185 --seed 2 --direct-seeds 5 --max-runtime 240 > gpurun_out/${T}_ttt_185.jsonl 2> gpurun_out/${T}_ttt_185.err; echo "ttt185 rc=$?"
cut -c1-220 gpurun_out/${T}_config5.jsonl gpurun_out/${T}_ttt_171.jsonl gpurun_out/${T}_ttt_185.jsonl
