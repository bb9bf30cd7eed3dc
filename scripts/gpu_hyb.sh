#!/bin/bash
# A/B of the restore-and-multiply half-1 register products (BS_RG_HYB=1, default) vs all-TMEM (0)
O=gpurun_out/hyb; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rgemv or prefill or more_than or numerics or smoke or dispatch or guard" > $O/tests.log 2>&1; echo tests=$?; tail -3 $O/tests.log
for args in "--batch 8" "--workload c5 --batch 8" "--workload c3_up" "--workload c3_down" "--batch 32"; do
  for h in 1 0; do
    BS_RG_HYB=$h timeout 300 python bench.py $args --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python scripts/bline.py | sed "s/^/hyb=$h /"
  done
done
