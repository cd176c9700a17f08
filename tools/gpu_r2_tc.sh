#!/bin/bash
# Evaluator iteration: probe + parity for the production evaluator, an A/B of
# build variants (SOKOL_LIB) on the length sweep, the bench, one ncu capture.
#   VARIANTS="libsokol_a.so libsokol_b.so" bash tools/gpu_r2_tc.sh
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-tc}
timeout 900 python -m pytest tests/test_gpu_evalprobe.py -x -q -k "fast or bounds or many or rejects" > gpurun_out/${T}_probe.log 2>&1; echo "probe rc=$?"; tail -2 gpurun_out/${T}_probe.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "fast" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/${T}_parity.log
for v in ${VARIANTS:-}; do
  SOKOL_LIB=$PWD/paper_2210_15962_b200/$v timeout 600 python tools/sweep.py --lengths ${LENGTHS:-101,201,255,301,449} --walk-factors 8 --seconds 1.0 > gpurun_out/${T}_sweep_$v.jsonl 2>&1
  echo "== $v"; cut -c1-160 gpurun_out/${T}_sweep_$v.jsonl
done
timeout 600 python tools/sweep.py --lengths ${LENGTHS:-101,201,255,301,449} --walk-factors 8 --seconds 1.0 > gpurun_out/${T}_sweep.jsonl 2>&1
echo "== libsokol.so"; cut -c1-160 gpurun_out/${T}_sweep.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; cut -c1-300 gpurun_out/${T}_bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/${T}_prof -f \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 65536 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
fi
