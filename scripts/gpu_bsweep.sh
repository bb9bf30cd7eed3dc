#!/bin/bash
# Batch sweep of the decode / prefill paths: c2 and c5 at B = 1..16 (AUTO dispatch), plus the
# prefill path forced at B = 2..12 (BS_FORCE_PREFILL) for the crossover.
for W in c2 c5; do
  for B in 1 2 3 4 5 6 8 10 12 16; do
    python bench.py --workload $W --batch $B --steps 1000 --warmup 20 --no-cpu-baseline
  done
done > gpurun_out/bsweep.jsonl 2> gpurun_out/bsweep.err
python scripts/bline.py < gpurun_out/bsweep.jsonl
for W in c2 c5; do
  for B in 2 4 8 12; do
    python bench.py --workload $W --batch $B --kernel prefill --steps 1000 --warmup 20 --no-cpu-baseline
  done
done > gpurun_out/bsweep_pf.jsonl 2>> gpurun_out/bsweep.err
python scripts/bline.py < gpurun_out/bsweep_pf.jsonl
