set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/c2.json 2>gpurun_out/c2.err; echo rc=$?
timeout 300 python bench.py --workload c5 --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/c5.json 2>gpurun_out/c5.err; echo rc=$?
timeout 300 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/c4.json 2>gpurun_out/c4.err; echo rc=$?
python - <<'P'
import json
for f in ("gpurun_out/c2.json", "gpurun_out/c5.json", "gpurun_out/c4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["value"], d["roofline"]["frac"], d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e)
P
timeout 300 python scripts/exp_timeline.py 2>&1 | head -12
