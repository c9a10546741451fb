python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider -x > gpurun_out/mp_r02b.log 2>&1; echo "mp pytest rc=$?"; tail -15 gpurun_out/mp_r02b.log
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_c1.py > gpurun_out/sanitizer_${tool}_r02b.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_r02b.log
done
