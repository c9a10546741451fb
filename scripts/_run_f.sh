python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gather.py -q -p no:cacheprovider -k "tc2_gather" -x > gpurun_out/tc2g_r02f.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/tc2g_r02f.log
for cfg in "c4 2 1e-5" "c3 2 1e-5" "c2 2 1e-4"; do
  timeout 300 python scripts/engine_ab.py $cfg 'pivots=8,l2_engine=3' 'pivots=8,l2_engine=6' 'pivots=8,l2_engine=4' 'pivots=8,l2_engine=1' 2>&1 | tail -4
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > /dev/null 2>&1; echo ncu_rc=$?
