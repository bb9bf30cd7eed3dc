#!/bin/bash
# final batch sweeps (AUTO and forced restore-and-multiply) + the b8 bench lines
O=gpurun_out/r02
mkdir -p $O
for W in c2 c5; do for B in 1 2 3 4 5 6 8 12 16 24 32 48; do
  timeout 300 python bench.py --workload $W --batch $B --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep.jsonl 2> $O/bsweep.err
./scripts/gpu_rg_final.sh
python scripts/bline.py < $O/bsweep.jsonl
