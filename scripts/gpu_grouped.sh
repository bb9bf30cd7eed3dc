# grouped decode launches: parity tests + C4 grouped vs per-matrix calls
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "grouped" > gpurun_out/pytest_grouped.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_grouped.log
timeout 300 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/c4_grouped.json 2>gpurun_out/c4_grouped.err; echo rc=$?
timeout 300 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline --no-group > gpurun_out/c4_single.json 2>gpurun_out/c4_single.err; echo rc=$?
cat gpurun_out/c4_grouped.json gpurun_out/c4_single.json; tail -5 gpurun_out/c4_grouped.err
