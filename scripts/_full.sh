python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/all_r02x.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/all_r02x.log
timeout 900 python bench.py > gpurun_out/bench_r02x.json 2> gpurun_out/bench_r02x.err; echo bench_rc=$?
