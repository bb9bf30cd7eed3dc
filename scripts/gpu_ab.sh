# A/B: parity with the candidate (BS_DECODE_DYN=1) + bench c2 for both
BS_DECODE_DYN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for r in 1 2; do for v in 0 1; do BS_DECODE_DYN=$v timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); print('v=$v', 'us/layer %.2f' % d['us_per_layer'], 'GB/s %.0f' % d['value'], 'kernel_us %.2f' % d['roofline']['kernel_us'], 'frac %.3f' % d['roofline']['frac'])"; done; done
