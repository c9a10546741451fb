# Full GPU pass of the current tree: build, every -m gpu test, the default bench line, smoke.
# usage (GPU box): bash scripts/_full.sh TAG
TAG=${1:-run}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/all_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/all_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_rc=$?
