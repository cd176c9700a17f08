#!/bin/bash
# A/B of build variants, interleaved to average clock/thermal drift:
#   VARIANTS="libsokol.so libsokol_x.so" LENGTHS=201,449 REPS=3 bash tools/gpu_ab_r2.sh
mkdir -p gpurun_out
T=${TAG:-ab}
for r in $(seq 1 ${REPS:-3}); do
  for v in ${VARIANTS}; do
    SOKOL_LIB=$PWD/paper_2210_15962_b200/$v timeout 300 python tools/sweep.py --lengths ${LENGTHS:-201} --walk-factors 8 --seconds ${SECS:-1.5} \
      | sed "s/^/{\"lib\": \"$v\", \"rep\": $r, \"pt\": /; s/$/}/" >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
  done
done
python - <<'PY'
import json, collections, os
T = os.environ.get("TAG", "ab")
d = collections.defaultdict(list)
for line in open(f"gpurun_out/{T}.jsonl"):
    try:
        r = json.loads(line)
    except Exception:
        continue
    d[(r["lib"], r["pt"]["L"])].append(r["pt"]["nse_per_s"])
for k in sorted(d):
    v = d[k]
    print(k, "n=%d mean=%.4g min=%.4g max=%.4g" % (len(v), sum(v) / len(v), min(v), max(v)))
PY
