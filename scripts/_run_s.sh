python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 300 python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 2>&1 | tail -1 | cut -c1-300
timeout 300 python scripts/engine_ab.py c3 2 1e-5 'pivots=1' 2>&1 | tail -1 | cut -c1-300
timeout 300 python scripts/engine_ab.py c2 2 1e-4 'pivots=8' 2>&1 | tail -1 | cut -c1-300
bash scripts/micro/build_prof.sh > gpurun_out/prof_build.log 2>&1; ENGINE=3 PIVOTS=8 bash scripts/micro/run_tc_prof.sh c4 1e-05 2>&1 | tail -9
