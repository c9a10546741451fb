#!/bin/bash
# per-kernel launch list of one join (engine_ab, warmup 2 + 5 steps) for a config: cfg norm hit opts
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ll.log 2>&1 || exit 1
for spec in "$@"; do
  set -- $spec
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$1_$2.csv python scripts/engine_ab.py $1 $2 $3 $4 > gpurun_out/ll_$1_$2.log 2>&1
  echo "$spec rc=$?"
done
