#!/bin/bash
# Projected 1/2/4/8-GPU device times from sequential shards on one GPU (diagnostic).
# usage: bash scripts/emulate_scaling.sh c3:1e-05 c5:1e-06
for spec in "${@:-c3:1e-05}"; do
  cfg=${spec%%:*}; hit=${spec##*:}
  for W in 1 2 4 8; do
    timeout 1500 python bench.py --config $cfg --norms 2 --hit $hit --steps ${STEPS:-3} --warmup 1 --emulate-ranks $W 2>&1 | tail -1
  done
done
