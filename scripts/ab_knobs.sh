#!/bin/bash
# A/B of environment knobs on bench configs.
# usage: CFGS="c3:1e-05 c4:1e-05" KNOBS="KGC_TC2=0,KGC_T2_PREFETCH=0 KGC_TC2=0,KGC_T2_PREFETCH=1" bash scripts/ab_knobs.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1 || { echo build failed; exit 1; }
for spec in ${CFGS}; do
  cfg=${spec%%:*}; hit=${spec##*:}
  for knob in ${KNOBS}; do
    st=${STEPS:-5}; [ $cfg == c5 ] && st=2
    tag=$(echo $knob | tr ',=' '__')
    env $(echo $knob | tr ',' ' ') timeout 900 python bench.py --config $cfg --norms ${NORMS:-2} --hit $hit --steps $st --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${cfg}_$tag.json 2>gpurun_out/ab_${cfg}_$tag.err
    python - $cfg $tag <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/ab_{c}_{v}.json"))
except Exception as e:
    print(c, v, "FAILED"); sys.exit(0)
tk = [k for k in d["kernels"] if "tiles" in k["kernel"]][0]
print("%s %-32s ms/step %8.3f value %.4g | %s %.3f ms %.1f TF/s frac %.3f clk %s" % (c, v, d["ms_per_step"], d["value"], tk["kernel"][:16], tk["ms"], tk.get("achieved", 0), tk.get("achieved", 0) / tk.get("peak", 1), d["clocks"]["sm_mhz"]))
PY
  done
done
