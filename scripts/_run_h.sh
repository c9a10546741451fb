python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
for cfg in "c4 2 1e-5" "c3 2 1e-5"; do
  timeout 300 python scripts/engine_ab.py $cfg 'pivots=8,l2_engine=6' 2>&1 | tail -1 | cut -c1-420
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02h.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > /dev/null 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify|mp_qkeys|pick_pivots|mp_keys|radix" -s 0 -c 12 -o gpurun_out/prof_r02h python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_r02h.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/prof_r02h.ncu-rep --page raw --csv > gpurun_out/prof_r02h_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02h.ncu-rep --page details --csv > gpurun_out/prof_r02h_details.csv 2>/dev/null
ls -la gpurun_out/prof_r02h*; sz=$(stat -c %s gpurun_out/prof_r02h.ncu-rep); if [ "$sz" -gt 25000000 ]; then rm -f gpurun_out/prof_r02h.ncu-rep; fi
