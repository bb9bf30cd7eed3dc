#!/bin/bash
# restore-and-multiply path: batch sweep of the forced kernel (C2, C5) and one ncu capture
O=gpurun_out/rg
mkdir -p $O
for W in c2 c5; do for B in 1 3 8 16 32; do
  timeout 300 python bench.py --workload $W --batch $B --kernel rgemv --steps 500 --warmup 10 --no-cpu-baseline
done; done > $O/rg.jsonl 2> $O/rg.err
python scripts/bline.py < $O/rg.jsonl
tail -3 $O/rg.err
CMD="python bench.py --workload c2 --batch 8 --kernel rgemv --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rgemv" -s 5 -c 1 -o $O/rg_c2 $CMD > $O/ncu.log 2>&1; echo ncu=$?
