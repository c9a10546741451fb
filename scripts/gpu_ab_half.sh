#!/bin/bash
# half-tile gathered L1 units: parity (debug build, KGC_GT_HALF=1) and A/B timing on c2 L1
mkdir -p gpurun_out
KGC_BUILD_EXPERIMENTS=1 python -c "from paper_2307_12059_b200 import _build; _build.build(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
KGC_GT_HALF=1 timeout 900 python -m pytest tests/test_gpu_gather.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
echo "base"; KGC_GT_VAR=0 timeout 300 python scripts/engine_ab.py c2 1 0.0001 'pivots=8' 2>&1 | tail -1
for V in ${VARS:-0 1 2 3}; do
  echo "half var $V"; KGC_GT_HALF=1 KGC_GT_VAR=$V timeout 300 python scripts/engine_ab.py c2 1 0.0001 'pivots=8' 2>&1 | tail -1
done
