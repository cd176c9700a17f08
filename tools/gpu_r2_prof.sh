#!/bin/bash
# one ncu --set full capture of the bench's walk kernel (65536 walks, L=201) for source-level analysis
mkdir -p gpurun_out
T=${TAG:-prof}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/${T}_prof -f \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 65536 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
