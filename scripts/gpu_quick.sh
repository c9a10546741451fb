#!/bin/bash
# quick loop: build, a pytest selection ($PYT, $PYK; SKIP_TESTS=1 skips), whole-join phases (engine_ab)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_q.log 2>&1 || { tail gpurun_out/build_q.log; exit 1; }
[ "${SKIP_TESTS:-0}" == "1" ] || timeout 1200 python -m pytest ${PYT:-tests/test_gpu_gather.py} -m gpu -q -x -p no:cacheprovider ${PYK} 2>&1 | tail -2
# configs: the script's arguments (one quoted "cfg norm hit opts" each), default c4 / c3 / c2
[ $# -eq 0 ] && set -- "c4 2 1e-05 pivots=64" "c3 2 1e-05 pivots=64" "c2 1 0.0001 pivots=32"
for c in "$@"; do
  echo "== $c"; timeout 600 python scripts/engine_ab.py $c 2>&1 | grep opts | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('total %.2f keys %.2f sort %.2f ranges %.2f stage %.2f tiles %.2f recheck %.2f' % (d['ms_total'], d['ms_keys'], d['ms_sort'], d['ms_ranges'], d['ms_stage'], d['ms_tiles'], d['ms_recheck']))"
done
