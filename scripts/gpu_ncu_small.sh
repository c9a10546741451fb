#!/bin/bash
# ncu --set full of the small K1-K3 / staging kernels (one launch each)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ns.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mp_qkeys_fact|mp_ent|mp_count" -s 3 -c 3 -o gpurun_out/prof_ns4 python scripts/engine_ab.py c4 2 1e-05 pivots=8 > gpurun_out/ncu_ns4.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stage_simt|gather_tails_block" -s 2 -c 2 -o gpurun_out/prof_ns2 python scripts/engine_ab.py c2 1 0.0001 pivots=8 > gpurun_out/ncu_ns2.log 2>&1; echo rc=$?
for t in ns4 ns2; do ncu -i gpurun_out/prof_$t.ncu-rep --page raw --csv > gpurun_out/prof_${t}_raw.csv 2>/dev/null; ncu -i gpurun_out/prof_$t.ncu-rep --page source --csv > gpurun_out/prof_${t}_src.csv 2>/dev/null; done
ls -la gpurun_out
