# parity + C2 bench (2 reps) of the default build
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline > gpurun_out/ab_$r.json 2> gpurun_out/ab_$r.err; python -c "
import json; d=json.load(open('gpurun_out/ab_$r.json')); print('rep $r', 'us/layer %.2f' % d['us_per_layer'], 'GB/s %.0f' % d['value'], 'kernel_us %.2f' % d['roofline']['kernel_us'], 'frac %.3f' % d['roofline']['frac'])"; done
