for v in "" nosttm nomma noexpand nosttm_nomma; do
  if [ -z "$v" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_$v.so"; fi
  env $L timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline > gpurun_out/exp_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/exp_$v.json')); print('${v:-baseline}', 'us/layer %.2f' % d['us_per_layer'], 'kernel_us %.2f' % d['roofline']['kernel_us'])"
done
