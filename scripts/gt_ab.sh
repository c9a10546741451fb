#!/bin/bash
# A/B of the gathered-tail kernel variants on c2 L1 (bench --norms 1), then one ncu --set full capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_gt.log 2>&1 || exit 1
for V in ${VARS:-0 1 2 3}; do
  KGC_GT_VAR=$V timeout 120 python bench.py --norms 1 --no-cpu --no-e2e > gpurun_out/gt_v$V.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/gt_v$V.json').read())
k=[k for k in d['kernels'] if 'achieved' in k][0]
print('var $V ms/step %.3f tiles %.3f ms frac %.3f' % (d['ms_per_step'], k['ms'], k['achieved']/k['peak']))"
done
if [ "${NCU:-1}" == "1" ]; then
  KGC_GT_VAR=${NCU_VAR:-0} timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiles_gather" -s 2 -c 1 -o gpurun_out/prof_gt python bench.py --norms 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_gt.log 2>&1
  echo "ncu rc=$?"
fi
