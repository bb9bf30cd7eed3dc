BS_DECODE_DYN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for v in dyn static; do
  case $v in dyn) L="BS_DECODE_DYN=1";; static) L="BS_DECODE_DYN=0";; esac
  env $L timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline > gpurun_out/rep_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/rep_$v.json')); print('$v', 'us/layer %.2f' % d['us_per_layer'], 'kernel_us %.2f' % d['roofline']['kernel_us'])"; done
