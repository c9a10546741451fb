#!/bin/bash
# One GPU round trip: build, parity tests, bench, launch list, ncu capture of the tile kernels.
# usage (under gpurun): bash scripts/gpu_check.sh [tag] [pytest-args]
TAG=${1:-dev}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench_rc=$?"; cat gpurun_out/bench_$TAG.json | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print('value %.4g ms/step %.3f roofline %s frac %.3f e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], (d['e2e'] or {}).get('value',0)))
  for k in d['kernels']: print('   %-45s %8.3f ms %s' % (k['kernel'], k['ms'], ('%.1f/%.1f %s' % (k['achieved'], k['peak'], k['unit'])) if 'achieved' in k else ''))
  print('   pruned', d['pruned_tile_fraction'], 'cand/res', d['candidates_per_result'], 'clocks', d['clocks'])
"
tail -2 gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" == "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS} > /dev/null 2>&1
  echo "ncu_launches_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-tiles_|verify}" -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-3} -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu_full_rc=$?"
  # export the raw metrics page here (gpurun copies back at most 64 MiB); keep the report only if small
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
  if [ -n "${SRC_KERNEL}" ]; then
    ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --kernel-name regex:"${SRC_KERNEL}" --launch-count 1 > gpurun_out/prof_${TAG}_src.csv 2>/dev/null
  fi
  sz=$(stat -c %s gpurun_out/prof_$TAG.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 25000000 ]; then rm -f gpurun_out/prof_$TAG.ncu-rep; fi
fi
