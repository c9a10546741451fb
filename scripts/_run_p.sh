python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_r02p.json 2> gpurun_out/bench_r02p.err; echo bench_rc=$?
tail -2 gpurun_out/bench_r02p.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02p.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > /dev/null 2>&1; echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tiles_tc2|verify|qkeys" -s 0 -c 3 -o gpurun_out/prof_r02p python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_r02p.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/prof_r02p.ncu-rep --page raw --csv > gpurun_out/prof_r02p_raw.csv 2>/dev/null
sz=$(stat -c %s gpurun_out/prof_r02p.ncu-rep); if [ "$sz" -gt 25000000 ]; then rm -f gpurun_out/prof_r02p.ncu-rep; fi
ls -la gpurun_out/ | tail -5
