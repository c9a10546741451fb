mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_tc2.log 2>&1 || { echo build failed; tail gpurun_out/build_tc2.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_parity.py -k "tc2 and not full_size" -x -q -p no:cacheprovider > gpurun_out/pytest_tc2.log 2>&1
echo "pytest_rc=$?"; tail -15 gpurun_out/pytest_tc2.log
