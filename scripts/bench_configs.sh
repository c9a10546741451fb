#!/bin/bash
# Extra bench lines for the large L2 configs (run under gpurun after gpu_check.sh).
for spec in "c3 1e-05" "c4 1e-05" ${EXTRA_CONFIGS}; do
  set -- $spec
  timeout 900 python bench.py --config $1 --norms 2 --hit $2 --steps ${STEPS:-5} --no-cpu ${BENCH_EXTRA} > gpurun_out/bench_$1_${TAG:-dev}.json 2>gpurun_out/bench_$1_${TAG:-dev}.err
  echo "$1 rc=$?"
  python - "$1" <<'PY'
import json, sys
c = sys.argv[1]
import os
d = json.load(open(f"gpurun_out/bench_{c}_{os.environ.get('TAG','dev')}.json"))
print("  %s value %.4g ms/step %.3f frac %.3f pruned %s cand/res %s e2e %s" % (c, d["value"], d["ms_per_step"], d["roofline"]["frac"],
      d["pruned_tile_fraction"], d["candidates_per_result"], (d.get("e2e") or {}).get("value")))
for k in d["kernels"]:
    print("     %-45s %8.3f ms" % (k["kernel"], k["ms"]))
PY
done
