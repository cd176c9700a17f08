#!/bin/bash
# probe + fast parity on libsokol.so, then an interleaved A/B against VARIANTS
mkdir -p gpurun_out
T=${TAG:-tcab}
timeout 900 python -m pytest tests/test_gpu_evalprobe.py -x -q -k "fast or bounds or many or rejects" > gpurun_out/${T}_probe.log 2>&1; echo "probe rc=$?"; tail -1 gpurun_out/${T}_probe.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "fast" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/${T}_parity.log
TAG=${T}_ab VARIANTS="libsokol.so ${VARIANTS}" LENGTHS=${LENGTHS:-201,301,449} REPS=${REPS:-3} bash tools/gpu_ab_r2.sh
