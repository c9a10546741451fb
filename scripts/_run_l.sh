python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 300 python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 2>&1 | tail -1 | cut -c1-330
timeout 300 python scripts/engine_ab.py c2 2 1e-4 'pivots=8' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
timeout 300 python scripts/engine_ab.py c2 1 1e-4 'pivots=8' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
timeout 300 python scripts/engine_ab.py c3 2 1e-4 'pivots=1' 2>&1 | tail -1 | cut -c1-330
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -p no:cacheprovider -x > gpurun_out/par_r02l.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/par_r02l.log
