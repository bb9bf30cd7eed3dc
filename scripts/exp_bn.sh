# prefill GEMM tile shapes: BN x MH per C3 matrix (BS_PREFILL_BN / BS_PREFILL_MH overrides)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k prefill 2>&1 | tail -1
for cfg in "0 0" "256 1" "128 1" "192 2" "224 2" "256 2"; do
  set -- $cfg
  for wl in c3_up c3_down; do
    BS_PREFILL_BN=$1 BS_PREFILL_MH=$2 timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bn_${wl}_$1_$2.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/bn_${wl}_$1_$2.json').read().strip().splitlines()[-1]); print('$wl', 'BN=$1 MH=$2', round(d['ms_per_step']*1e3,1), 'us step', round(d['roofline']['kernel_us'],1), 'us gemm')"
  done
done
