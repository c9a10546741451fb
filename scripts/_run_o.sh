python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
for cfg in c4 c3; do for sp in 0 2; do
  timeout 600 python bench.py --config $cfg --emulate-ranks 8 --split $sp --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg split $sp', [round(x,2) for x in d['shard_ms']], 'proj', round(d['projected_ms_per_step'],2))"
done; done
timeout 600 python bench.py --config c4 --emulate-ranks 1 --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 W1', d['shard_ms'])"
timeout 600 python bench.py --config c3 --emulate-ranks 1 --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 W1', d['shard_ms'])"
timeout 900 python bench.py --config c5 --emulate-ranks 8 --split 2 --steps 1 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 split 2', [round(x,1) for x in d['shard_ms']])"
timeout 900 python bench.py --config c5 --emulate-ranks 8 --split 0 --steps 1 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 split 0', [round(x,1) for x in d['shard_ms']])"
