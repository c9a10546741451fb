python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -p no:cacheprovider -x -k "pivot or offset or c5 or concurrent or keys" > gpurun_out/keys_r02i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/keys_r02i.log
timeout 300 python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 2>&1 | tail -1 | cut -c1-300
timeout 300 python scripts/engine_ab.py c2 1 1e-4 'pivots=8' 2>&1 | tail -1 | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify|qkeys" -s 0 -c 3 -o gpurun_out/prof_r02i python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_r02i.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/prof_r02i.ncu-rep --page raw --csv > gpurun_out/prof_r02i_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02i.ncu-rep --page source --csv --kernel-name regex:verify --launch-count 1 > gpurun_out/prof_r02i_src_verify.csv 2>/dev/null
ls -la gpurun_out/prof_r02i*; sz=$(stat -c %s gpurun_out/prof_r02i.ncu-rep); if [ "$sz" -gt 25000000 ]; then rm -f gpurun_out/prof_r02i.ncu-rep; fi
