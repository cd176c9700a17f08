#!/bin/bash
# parity of the in-tree build (fast setups, evaluator probe) and an interleaved A/B against other builds:
#   TAG=nc2 VARIANTS="libsokol_head.so libsokol.so" LENGTHS=201,449 bash tools/gpu_r2_nc.sh
mkdir -p gpurun_out
T=${TAG:-nc}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_evalprobe.py -x -q -k "fast or probe or evalprobe" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/${T}_parity.log
TAG=${T}_ab VARIANTS="${VARIANTS:-libsokol_head.so libsokol.so}" LENGTHS=${LENGTHS:-201,449} REPS=${REPS:-3} bash tools/gpu_ab_r2.sh
