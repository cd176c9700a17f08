#!/bin/bash
# racecheck in slices (one length per process, so each fits the timeout), plus a parity/perf check of libsokol.so
mkdir -p gpurun_out
T=${TAG:-race}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evalprobe.py tests/test_gpu_configs.py -x -q > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/${T}_parity.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.json 2>&1; cut -c1-200 gpurun_out/${T}_bench.json
for L in ${LENGTHS:-449}; do
  SANITIZE_LENGTHS=$L SANITIZE_W=${SANITIZE_W:-4} timeout ${RT:-1500} compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py \
    > gpurun_out/${T}_racecheck_L$L.log 2>&1; echo "racecheck L=$L rc=$?"; tail -2 gpurun_out/${T}_racecheck_L$L.log
done
