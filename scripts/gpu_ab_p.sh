# A/B of decode geometries: default (R4 P1), R2 P2 (scripts/libbitstack_p2.so), R2 P1
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pt_def.log 2>&1; echo def_rc=$?; tail -2 gpurun_out/pt_def.log
BITSTACK_LIB=$PWD/scripts/libbitstack_p2.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pt_p2.log 2>&1; echo p2_rc=$?; tail -2 gpurun_out/pt_p2.log
for v in def p2 r2; do
  if [ $v = def ]; then export BITSTACK_LIB=; else export BITSTACK_LIB=$PWD/scripts/libbitstack_$v.so; fi
  [ -z "$BITSTACK_LIB" ] && unset BITSTACK_LIB
  for wl in c2 c5; do timeout 300 python bench.py --workload $wl --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/ab_${v}_$wl.json 2>/dev/null; done
  timeout 300 python bench.py --workload c2 --batch 2 --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/ab_${v}_c2b2.json 2>/dev/null
  timeout 300 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${v}_c4.json 2>/dev/null
done
python - <<'P'
import json
for v in ("def", "p2", "r2"):
    for wl in ("c2", "c2b2", "c5", "c4"):
        f = f"gpurun_out/ab_{v}_{wl}.json"
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            print(v, wl, round(d["ms_per_step"] * 1e3, 2), "us", round(d["value"]), d["roofline"]["frac"])
        except Exception as e:
            print(v, wl, "ERR", e)
P
