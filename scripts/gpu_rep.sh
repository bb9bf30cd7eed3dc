# A/B on one box: default build vs scripts/libbitstack_prev.so, 2 reps each
for r in 1 2; do for v in cur prev; do
  if [ "$v" = "cur" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_prev.so"; fi
  env $L timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline > gpurun_out/rep_$v$r.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/rep_$v$r.json')); print('$v $r', 'us/layer %.2f' % d['us_per_layer'], 'kernel_us %.2f' % d['roofline']['kernel_us'])"; done; done
