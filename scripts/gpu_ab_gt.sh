#!/bin/bash
# A/B of the gathered-tail L1 kernel variants (debug build: KGC_GT_VAR) on c2 L1, per-phase device times.
mkdir -p gpurun_out
KGC_BUILD_EXPERIMENTS=1 python -c "from paper_2307_12059_b200 import _build; _build.build(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
for V in ${VARS:-0 4 5 6 7 8 9 10 11 12}; do
  echo "var $V"; KGC_GT_VAR=$V timeout 300 python scripts/engine_ab.py c2 1 0.0001 'pivots=8' 2>&1 | tail -1
done
