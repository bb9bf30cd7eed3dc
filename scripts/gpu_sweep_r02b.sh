#!/bin/bash
# AUTO batch sweep after the restore-and-multiply dispatch (decode <= 5, rgemv 6..32, prefill > 32),
# plus one ncu capture of the rgemv kernel and the default C2 line
O=gpurun_out/r02b
mkdir -p $O
for W in c2 c5; do for B in 1 2 3 4 5 6 8 12 16 24 32 48; do
  timeout 300 python bench.py --workload $W --batch $B --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep.jsonl 2> $O/bsweep.err
python scripts/bline.py < $O/bsweep.jsonl
timeout 300 python bench.py --steps 20000 --warmup 200 > $O/bench_c2.json 2> $O/bench_c2.err; python scripts/bline.py < $O/bench_c2.json
CMD="python bench.py --workload c2 --batch 8 --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rgemv" -s 5 -c 1 -o $O/rg_c2 $CMD > $O/ncu.log 2>&1; echo ncu=$?
