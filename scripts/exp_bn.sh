timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for wl in c3_up c3_down; do
  timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/pf_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf_$wl.json')); print('$wl', 'us/step %.1f' % (d['ms_per_step']*1e3), 'gemm_us %.1f' % d['roofline']['kernel_us'], 'TF/s %.0f' % d['roofline']['achieved'], 'value %.0f' % d['value'])"
done
