#!/bin/bash
# the slow sanitizer slices on their own: synccheck on the default workload, racecheck at L=1023 (short walks)
mkdir -p gpurun_out
T=${TAG:-san}
SANITIZE_W=8 timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/${T}_sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/${T}_sanitize_synccheck.log
SANITIZE_LENGTHS=1023 SANITIZE_LAYOUTS=2 SANITIZE_W=2 SANITIZE_WF=1 timeout 2700 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/${T}_sanitize_racecheck_1023.log 2>&1; echo "racecheck 1023 rc=$?"; tail -3 gpurun_out/${T}_sanitize_racecheck_1023.log
