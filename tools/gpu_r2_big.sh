#!/bin/bash
# EvalTC for L <= 1023 (build variant libsokol_big.so): parity at the long lengths and an A/B against libsokol.so
mkdir -p gpurun_out
T=${TAG:-big}
export SOKOL_LIB=$PWD/paper_2210_15962_b200/libsokol_big.so
timeout 1200 python -m pytest tests/test_gpu_evalprobe.py tests/test_gpu_parity.py -x -q -k "fast and (513 or 769 or 1021 or 1023 or 511 or 385 or 1023)" > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/${T}_parity.log
unset SOKOL_LIB
TAG=${T}_ab VARIANTS="libsokol.so libsokol_big.so" LENGTHS=201,513,769,1023 REPS=2 bash tools/gpu_ab_r2.sh
