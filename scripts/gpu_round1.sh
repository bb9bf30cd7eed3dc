# Round-1 GPU evidence: full GPU tests, the default bench line, the ncu launch list of the
# bench command and one --set full capture of each kernel of the decode pair.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --sweep > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_r01.json
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_f8|zq_kernel" -s 40 -c 2 -o gpurun_out/decode_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
tail -3 gpurun_out/ncu_full.log
