#!/bin/bash
# Round-2 evidence pass on the production libsokol.so: smoke, every GPU test,
# the bench (native + reference arms), an ncu launch list and one ncu --set
# full capture of the bench kernel, then compute-sanitizer (memcheck,
# racecheck, synccheck) on tools/sanitize.py.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${T}_smi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${T}_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/${T}_bench_ref.json
timeout 900 python tools/sweep.py --lengths 27,101,121,151,171,201,223,255,257,301,401,449,511,1023 --walk-factors 8 --seconds 1.5 > gpurun_out/${T}_sweep.jsonl 2>&1; echo "sweep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:saw_walk_kernel -c 1 -o gpurun_out/${T}_prof -f \
    python bench.py --steps 1 --warmup 0 --walkers-per-gpu 65536 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
if [ "${SANITIZE:-1}" = "1" ]; then
for tool in memcheck synccheck racecheck; do
  SANITIZE_W=${SANITIZE_W:-8} timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py \
    > gpurun_out/${T}_sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/${T}_sanitize_$tool.log
done
fi
if [ "${SANITIZE_LONG:-0}" = "1" ]; then
for tool in memcheck racecheck; do
  SANITIZE_LENGTHS=513,1023 SANITIZE_LAYOUTS=2,3 SANITIZE_W=2 SANITIZE_WF=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py \
    > gpurun_out/${T}_sanitize_long_$tool.log 2>&1; echo "$tool (L=513,1023) rc=$?"; tail -2 gpurun_out/${T}_sanitize_long_$tool.log
done
fi
