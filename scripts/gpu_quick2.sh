timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for b in 1 2 4; do timeout 300 python bench.py --workload c2 --batch $b --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q_c2b$b.json 2>/dev/null; done
timeout 300 python bench.py --workload c5 --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q_c5.json 2>/dev/null
BITSTACK_LIB=$PWD/scripts/libbitstack_base.so timeout 300 python bench.py --workload c2 --batch 2 --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q_base_c2b2.json 2>/dev/null
python - <<'P'
import json, glob
for f in sorted(glob.glob("gpurun_out/q_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, f"{d['ms_per_step']*1e3:.2f}us", round(d["value"]), round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(f, "ERR", e)
P
