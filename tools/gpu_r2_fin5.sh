#!/bin/bash
# final evidence pass: gpu_r2_final.sh (smoke, GPU suite, bench both arms, sweep, ncu) + memcheck and short racecheck
T=${TAG:-fin5}
TAG=$T SANITIZE=0 SANITIZE_LONG=0 bash tools/gpu_r2_final.sh
SANITIZE_W=8 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/${T}_sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/${T}_sanitize_memcheck.log
SANITIZE_LENGTHS=27,201 SANITIZE_W=4 SANITIZE_WF=2 timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/${T}_sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/${T}_sanitize_racecheck.log
