for v in base nosttm_nomma noall; do
  if [ "$v" = "base" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_$v.so"; fi
  env $L timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline > gpurun_out/exp_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/exp_$v.json')); print('$v', 'us/layer %.2f' % d['us_per_layer'], 'kernel_us %.2f' % d['roofline']['kernel_us'])"
done
for n in 1 4; do
  env BITSTACK_LIB=scripts/libbitstack_noall.so timeout 300 python bench.py --n $n --steps 3000 --warmup 50 --no-cpu-baseline > gpurun_out/exp_n$n.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/exp_n$n.json')); print('noall n=$n', 'us/layer %.2f' % d['us_per_layer'], 'kernel_us %.2f' % d['roofline']['kernel_us'])"
done
