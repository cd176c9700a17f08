#!/bin/bash
# parity of a build variant (SOKOL_LIB) on the fast setups, then an interleaved A/B against libsokol.so
mkdir -p gpurun_out
T=${TAG:-var}
SOKOL_LIB=$PWD/paper_2210_15962_b200/${VAR} timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "fast" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/${T}_parity.log
TAG=${T}_ab VARIANTS="libsokol.so ${VAR}" LENGTHS=${LENGTHS:-201,449} REPS=${REPS:-3} bash tools/gpu_ab_r2.sh
