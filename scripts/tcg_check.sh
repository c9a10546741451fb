#!/bin/bash
# Gathered tensor-core engine: its parity tests, then c2 / c3 / c4 L2 bench A/B (contiguous vs gathered).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_tcg.log 2>&1 || { tail gpurun_out/build_tcg.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gather.py -q -x -p no:cacheprovider --timeout 90 -k "tc_gather" > gpurun_out/pt_tcg.log 2>&1
echo "tcg tests rc=$?"; tail -15 gpurun_out/pt_tcg.log
for CFG in ${CFGS:-c2:1e-4 c3:1e-5 c4:1e-5}; do
  C=${CFG%%:*}; H=${CFG##*:}
  for G in 0 1; do
    KGC_GATHER_TC=$G timeout 300 python bench.py --config $C --hit $H --norms 2 --pivots 8 --no-cpu --no-e2e > gpurun_out/tcg_${C}_$G.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/tcg_${C}_$G.json').read())
k=[k for k in d['kernels'] if 'achieved' in k][0]
print('$C gather=$G ms/step %.3f value %.4g tiles %.3f ms %s' % (d['ms_per_step'], d['value'], k['ms'], k['kernel']))" 2>&1 | tail -1
  done
done
