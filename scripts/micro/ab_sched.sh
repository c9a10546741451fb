python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for sc in 0 1; do for c in c2 c3; do
 KGC_SCHED_TC=$sc timeout 600 python bench.py --config $c --norms 2 --hit $([ $c == c2 ] && echo 1e-4 || echo 1e-05) --steps 5 --no-cpu --no-e2e > gpurun_out/ab_${c}_$sc.json 2>&1
 python -c "
import json; d=json.load(open('gpurun_out/ab_${c}_$sc.json')); print('$c sched $sc', [ (k['kernel'][:14], round(k['ms'],3)) for k in d['kernels'] if 'tiles' in k['kernel']])"
 KGC_SCHED_TC=$sc timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:tiles_tc -c 1 python bench.py --config $c --norms 2 --hit $([ $c == c2 ] && echo 1e-4 || echo 1e-05) --steps 1 --warmup 0 --no-cpu --no-e2e 2>&1 | grep -E "^\s+(gpu__|lts__|sm__|l1tex|dram)" 
done; done
