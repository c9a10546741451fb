set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k1.log 2>&1 || { tail gpurun_out/build_k1.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_stress.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_k1.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_k1.log
timeout 600 python bench.py --no-extras --no-cpu > gpurun_out/bench_k1.json 2> gpurun_out/bench_k1.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_k1.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], [(k['kernel'][:30], round(k['ms'],3)) for k in d['kernels']])
PY
cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 l1_inner.cu -o /tmp/l1_inner && /tmp/l1_inner; cd ../..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiles_gather -s 1 -c 1 -o gpurun_out/prof_l1 python bench.py --config c2 --no-extras --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_l1.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/prof_l1.ncu-rep --page raw --csv > gpurun_out/prof_l1_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_l1.ncu-rep --page source --csv --kernel-name regex:tiles_gather --launch-count 1 > gpurun_out/prof_l1_src.csv 2>/dev/null
ncu -i gpurun_out/prof_l1.ncu-rep --page details --csv > gpurun_out/prof_l1_details.csv 2>/dev/null
ls -la gpurun_out/
