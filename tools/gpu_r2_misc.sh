#!/bin/bash
# racecheck at L=449 with short walks, the multi-process bench paths, and an A/B of warps-per-block variants
mkdir -p gpurun_out
T=${TAG:-misc}
SANITIZE_LENGTHS=449 SANITIZE_W=2 SANITIZE_WF=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py \
  > gpurun_out/${T}_racecheck_L449.log 2>&1; echo "racecheck L=449 rc=$?"; tail -3 gpurun_out/${T}_racecheck_L449.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${T}_bench_torchrun1.json 2> gpurun_out/${T}_bench_torchrun1.err; echo "torchrun1 rc=$?"; cut -c1-200 gpurun_out/${T}_bench_torchrun1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu-baseline --walkers-per-gpu 262144 \
  > gpurun_out/${T}_bench_gloo2.json 2> gpurun_out/${T}_bench_gloo2.err; echo "gloo2 rc=$?"; cut -c1-200 gpurun_out/${T}_bench_gloo2.json
TAG=${T}_ab VARIANTS="${VARIANTS}" LENGTHS=201 REPS=3 bash tools/gpu_ab_r2.sh
