#!/bin/bash
# Swap each scripts/variants/lib_<name>.so in as the package library and time the bench
# workloads.  Usage: scripts/run_variants.sh "base nocp" "c2 c5"
cd "$(dirname "$0")/.."
LIB=paper_2410_23918_b200/libbitstack.so
cp $LIB /tmp/lib_orig.so
for v in $1; do
  cp scripts/variants/lib_$v.so $LIB
  for w in $2; do
    steps=2000; [ "$w" = c5 ] && steps=300; [ "$w" = c4 ] && steps=100
    python bench.py --workload $w --steps $steps --warmup 20 --no-cpu-baseline ${EXTRA} 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('%-8s %-4s us/step %8.2f frac %.3f' % ('$v', '$w', d['ms_per_step']*1e3, d['roofline']['frac']))"
  done
done
cp /tmp/lib_orig.so $LIB
