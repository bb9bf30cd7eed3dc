set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for v in new base; do
  if [ $v = new ]; then unset BITSTACK_LIB; else export BITSTACK_LIB=$PWD/scripts/libbitstack_base.so; fi
  for wl in c2 c5; do timeout 300 python bench.py --workload $wl --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/z_${v}_$wl.json 2>/dev/null; done
  timeout 300 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/z_${v}_c4.json 2>/dev/null
done
unset BITSTACK_LIB
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_kernel|decode_f8i" -c 200 --csv --log-file gpurun_out/launches_zq.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
python - <<'P'
import json, glob
for f in sorted(glob.glob("gpurun_out/z_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, f"{d['ms_per_step']*1e3:.2f}us", round(d["value"]), round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(f, "ERR", e)
P
