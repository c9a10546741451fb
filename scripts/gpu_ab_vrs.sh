#!/bin/bash
# relation rows in shared memory for the re-check (KGC_VRS, debug build): parity + A/B
mkdir -p gpurun_out
KGC_BUILD_EXPERIMENTS=1 python -c "from paper_2307_12059_b200 import _build; _build.build(force=True)" > gpurun_out/build_vrs.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for c in "c4 2 1e-05 pivots=64" "c2 2 0.0001 pivots=32" "c2 1 0.0001 pivots=32"; do
  for V in 0 1; do
    echo "== $c VRS=$V"; KGC_VRS=$V timeout 600 python scripts/engine_ab.py $c 2>&1 | grep opts | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('total %.2f recheck %.3f results %d' % (d['ms_total'], d['ms_recheck'], d['results']))"
  done
done
