python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"verify" -s 1 -c 1 -o gpurun_out/prof_r02m python scripts/engine_ab.py c4 2 1e-5 'pivots=8' > gpurun_out/ncu_r02m.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/prof_r02m.ncu-rep --page raw --csv > gpurun_out/prof_r02m_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02m.ncu-rep --page details --csv > gpurun_out/prof_r02m_details.csv 2>/dev/null
ncu -i gpurun_out/prof_r02m.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r02m_sass.csv 2>/dev/null
ls -la gpurun_out/prof_r02m*
