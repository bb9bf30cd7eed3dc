# quick iteration: parity tests, bench, ncu full capture of the decode kernel (n=16 and n=1)
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "not full_size" 2>&1 | tail -3
timeout 600 python bench.py --sweep > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
CMD="python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-graph"
if [ "$1" = "ncu" ]; then
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 20 -c 1 -o gpurun_out/dec_n16 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
CMD1="python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-graph --n 1"
timeout 300 $CMD1 > gpurun_out/plain1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 20 -c 1 -o gpurun_out/dec_n1 $CMD1 > gpurun_out/ncu_full1.log 2>&1; echo ncu1_rc=$?
fi
