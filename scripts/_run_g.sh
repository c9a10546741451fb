python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gather.py -q -p no:cacheprovider -k "tc2_gather or tc_gather" -x > gpurun_out/tcg_r02g.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/tcg_r02g.log
for cfg in "c4 2 1e-5" "c3 2 1e-5" "c2 2 1e-4"; do
  timeout 300 python scripts/engine_ab.py $cfg 'pivots=8,l2_engine=3' 'pivots=8,l2_engine=6' 'pivots=8,l2_engine=4' 2>&1 | tail -3
done
