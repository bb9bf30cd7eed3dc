#!/bin/bash
# restore-and-multiply lines with the TMEM-read roofline (bench.py "bound": "tmem")
O=gpurun_out/r02
mkdir -p $O
for W in c2 c5; do for B in 1 3 8 16 32; do
  timeout 300 python bench.py --workload $W --batch $B --kernel rgemv --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep_rgemv.jsonl 2> $O/bsweep_rgemv.err
for W in c2 c5; do timeout 300 python bench.py --workload $W --batch 8 --steps 1000 --warmup 20; done > $O/bench_rgemv_b8.jsonl 2>> $O/bsweep_rgemv.err
python scripts/bline.py < $O/bsweep_rgemv.jsonl
python -c "
import json
for l in open('$O/bench_rgemv_b8.jsonl'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'][:12], d['ms_per_step']*1e3, r['bound'], round(r['frac'],3), 'issue', round(r.get('issue_frac',0),3))
"
