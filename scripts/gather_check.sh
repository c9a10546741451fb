#!/bin/bash
# Gathered-tail engine round trip: build, its parity tests, the full GPU suite, bench A/B against contiguous tiles.
TAG=${1:-g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gather.py -q -x -p no:cacheprovider > gpurun_out/pytest_gather_$TAG.log 2>&1
echo "gather_rc=$?"; tail -15 gpurun_out/pytest_gather_$TAG.log
if [ "${FULL:-1}" == "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest_rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
fi
for G in 1 0; do
  KGC_GATHER=$G timeout 600 python bench.py --no-cpu > gpurun_out/bench_${TAG}_g$G.json 2> gpurun_out/bench_${TAG}_g$G.err
  echo "bench KGC_GATHER=$G rc=$?"
  python - gpurun_out/bench_${TAG}_g$G.json <<'PY'
import json,sys
for l in open(sys.argv[1]):
  d=json.loads(l); print('value %.4g ms/step %.3f roofline %s frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac']))
  for k in d['kernels']: print('   %-45s %8.3f ms %s' % (k['kernel'], k['ms'], ('%.1f/%.1f %s' % (k['achieved'], k['peak'], k['unit'])) if 'achieved' in k else ''))
PY
done
