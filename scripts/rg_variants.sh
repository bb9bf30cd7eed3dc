cd /root/repo
LIB=paper_2410_23918_b200/libbitstack.so
cp $LIB /tmp/lib_orig.so
for v in ${VARS:-base rg32 rgnoapply rgnocopy}; do
  cp scripts/variants/lib_$v.so $LIB
  for W in c2 c5; do
  python bench.py --workload $W --batch 8 --kernel rgemv --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('%-10s %s us/step %8.2f' % ('$v', '$W', d['ms_per_step']*1e3))"
  done
done
cp /tmp/lib_orig.so $LIB
