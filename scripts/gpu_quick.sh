#!/bin/bash
# quick A/B: GPU parity subset, then C2 / C5 / C4 / C2 B=2,8 bench lines
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or numerics or fuzz" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
( python bench.py --steps 5000 --warmup 50 --no-cpu-baseline --sweep
  python bench.py --workload c5 --steps 1000 --warmup 20 --no-cpu-baseline
  python bench.py --workload c4 --steps 200 --warmup 5 --no-cpu-baseline
  python bench.py --batch 2 --steps 2000 --warmup 20 --no-cpu-baseline
  python bench.py --batch 8 --steps 2000 --warmup 20 --no-cpu-baseline
  python bench.py --workload c5 --shard 8 --steps 2000 --warmup 20 --no-cpu-baseline ) > gpurun_out/quick.jsonl 2> gpurun_out/quick.err
python scripts/bline.py < gpurun_out/quick.jsonl
python -c "
import json
for l in open('gpurun_out/quick.jsonl'):
    d=json.loads(l)
    if 'n_sweep' in d: print('n sweep us', {k: round(v['us_per_layer'],1) for k,v in d['n_sweep'].items()})
"
