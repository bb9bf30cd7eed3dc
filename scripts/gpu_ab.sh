# parity of the default decode path + bench c2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline > gpurun_out/ab_0.json 2> gpurun_out/ab_0.err; echo "rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/ab_0.json')); print('us/layer %.2f' % d['us_per_layer'], 'GB/s %.0f' % d['value'], 'kernel_us %.2f' % d['roofline']['kernel_us'], 'frac %.3f' % d['roofline']['frac'])"
