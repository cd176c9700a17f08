#!/bin/bash
# Round-2 parity pass: new config / probe / multirank tests, the full GPU
# suite, then compute-sanitizer (memcheck, racecheck, synccheck) on tools/sanitize.py.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_evalprobe.py tests/test_gpu_configs.py tests/test_gpu_multirank.py -x -q \
  > gpurun_out/r2_new_tests.log 2>&1; echo "new tests rc=$?"
tail -5 gpurun_out/r2_new_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu_full.log 2>&1; echo "full gpu rc=$?"
tail -3 gpurun_out/r2_pytest_gpu_full.log
if [ "${SKIP_SANITIZE:-0}" = "0" ]; then
for tool in memcheck racecheck synccheck; do
  SANITIZE_W=32 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py \
    > gpurun_out/r2_sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -3 gpurun_out/r2_sanitize_$tool.log
done
fi
