#!/bin/bash
# verify_rows (8 lanes per candidate) vs the staged lane-per-candidate kernel: parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_v.log 2>&1 || { tail gpurun_out/build_v.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_se.py tests/test_gpu_topk.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
KGC_BUILD_EXPERIMENTS=1 python -c "from paper_2307_12059_b200 import _build; _build.build(force=True)" > gpurun_out/build_v2.log 2>&1 || exit 1
for c in "c4 2 1e-05 pivots=32" "c3 2 0.0001 pivots=24" "c2 2 0.0001 pivots=24" "c2 1 0.0001 pivots=24"; do
  for V in 0 1; do
    echo "== $c VROWS=$V"; KGC_VROWS=$V timeout 600 python scripts/engine_ab.py $c 2>&1 | grep opts | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('total %.2f recheck %.3f results %d cands %d' % (d['ms_total'], d['ms_recheck'], d['results'], d['candidates']))"
  done
done
