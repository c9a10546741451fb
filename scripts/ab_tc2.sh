#!/bin/bash
# A/B of the 1-CTA and CTA-pair tensor-core engines on the large L2 configs (KGC_TC2 = 0 / 1).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1 || { echo build failed; exit 1; }
for spec in ${CFGS:-c3:1e-05 c4:1e-05 c5:1e-06}; do
  cfg=${spec%%:*}; hit=${spec##*:}
  for v in 0 1; do
    st=${STEPS:-5}; [ $cfg == c5 ] && st=2
    KGC_TC2=$v timeout 900 python bench.py --config $cfg --norms 2 --hit $hit --steps $st --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${cfg}_$v.json 2>gpurun_out/ab_${cfg}_$v.err
    python - $cfg $v <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/ab_{c}_{v}.json"))
tk = [k for k in d["kernels"] if "tiles" in k["kernel"]][0]
print("%s tc2=%s ms/step %.3f value %.4g | %s %.3f ms %.1f TF/s frac %.3f" % (c, v, d["ms_per_step"], d["value"], tk["kernel"][:16], tk["ms"], tk.get("achieved", 0), tk.get("achieved", 0) / tk.get("peak", 1)))
PY
  done
done
