set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; echo bench rc=$?
tail -3 gpurun_out/r2_pytest_gpu.log; cat gpurun_out/r2_bench0.json
