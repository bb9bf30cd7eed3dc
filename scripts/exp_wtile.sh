# wtile G=2 (library default) vs G=4 (scripts/libbitstack_g4.so): prefill parity + c3 bench
BITSTACK_LIB=scripts/libbitstack_g4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k prefill 2>&1 | tail -2
for v in base g4; do
  if [ "$v" = "base" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_$v.so"; fi
  for wl in c3_up c3_down; do
    env $L timeout 300 python bench.py --workload $wl --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/w_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/w_${v}_$wl.json')); print('$v $wl', 'us/step %.1f' % (d['ms_per_step']*1e3), 'value %.1f' % d['value'], 'gemm_us %.1f' % d['roofline']['kernel_us'])"
  done
done
