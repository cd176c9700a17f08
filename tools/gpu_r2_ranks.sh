#!/bin/bash
# the multi-rank bench paths on one GPU: torchrun with NCCL at world size 1, and 2 gloo ranks sharing the GPU
mkdir -p gpurun_out
T=${TAG:-ranks}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${T}_bench_torchrun1.json 2> gpurun_out/${T}_bench_torchrun1.err; echo "torchrun1 rc=$?"; cut -c1-200 gpurun_out/${T}_bench_torchrun1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu-baseline --walkers-per-gpu 262144 \
  > gpurun_out/${T}_bench_gloo2.json 2> gpurun_out/${T}_bench_gloo2.err; echo "gloo2 rc=$?"; cut -c1-200 gpurun_out/${T}_bench_gloo2.json
