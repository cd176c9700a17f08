#!/bin/bash
# visited-set layouts with the round-2 evaluator, interleaved
mkdir -p gpurun_out
T=${TAG:-lay}
for r in 1 2 3; do
  for lay in 1 2 3; do
    SK_SWEEP_LAYOUT=$lay timeout 300 python tools/sweep.py --lengths ${LENGTHS:-201,301} --walk-factors 8 --seconds 1.5 \
      | sed "s/^/{\"layout\": $lay, \"rep\": $r, \"pt\": /; s/$/}/" >> gpurun_out/${T}.jsonl
  done
done
python - <<'PY'
import json, collections, os
d = collections.defaultdict(list)
for line in open("gpurun_out/" + os.environ.get("TAG", "lay") + ".jsonl"):
    r = json.loads(line); d[(r["layout"], r["pt"]["L"])].append((r["pt"]["nse_per_s"], r["pt"]["resident"]))
for k in sorted(d):
    v = [x[0] for x in d[k]]
    print(k, "resident", d[k][0][1], "mean %.4g max %.4g" % (sum(v) / len(v), max(v)))
PY
