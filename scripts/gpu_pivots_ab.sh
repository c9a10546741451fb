#!/bin/bash
# pivots A/B (whole join phases, engine_ab) + parity of the many-pivot paths
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pv.log 2>&1 || { tail gpurun_out/build_pv.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gather.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for c in "c4 2 1e-05" "c5 2 1e-06" "c3 2 1e-05" "c2 2 0.0001" "c2 1 0.0001"; do
  echo "== $c"; timeout 600 python scripts/engine_ab.py $c ${PVS:-pivots=8 pivots=16 pivots=24 pivots=32} 2>&1 | grep opts | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['opts'], 'total %.2f keys %.2f sort %.2f ranges %.2f stage %.2f tiles %.2f recheck %.2f tilefrac %.4f gfrac %.4f' % (d['ms_total'], d['ms_keys'], d['ms_sort'], d['ms_ranges'], d['ms_stage'], d['ms_tiles'], d['ms_recheck'], d['tile_pair_frac'], d['gathered_pair_frac']))"
done
