# Round-1 GPU evidence: full GPU tests, the default bench line (+ C5, C4, load, prefill lines),
# the ncu launch lists of the bench commands and --set full captures of the dominant kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --sweep > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_r01.json
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python bench.py --workload c5 --steps 2000 --warmup 20 > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err; echo c5_rc=$?
timeout 300 python bench.py --workload c4 --steps 200 --warmup 5 > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo c4_rc=$?
timeout 300 python bench.py --workload c4 --steps 200 --warmup 5 --no-group --no-cpu-baseline > gpurun_out/bench_c4_ungrouped.json 2>/dev/null; echo c4u_rc=$?
timeout 300 python bench.py --workload load --steps 10 --warmup 3 > gpurun_out/bench_load.json 2>gpurun_out/bench_load.err; echo load_rc=$?
timeout 300 python bench.py --workload compress --steps 5 --warmup 2 > gpurun_out/bench_compress.json 2>gpurun_out/bench_compress.err; echo compress_rc=$?
for b in 2 4 8 16; do timeout 300 python bench.py --batch $b --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c2_b$b.json 2>/dev/null; done
for wl in c3_up c3_down; do timeout 300 python bench.py --workload $wl --steps 300 --warmup 5 > gpurun_out/pf_$wl.json 2>gpurun_out/pf_$wl.err; echo pf_rc=$?; done
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_kernel|decode_f8i" -c 200 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_f8|zq_kernel" -s 40 -c 2 -o gpurun_out/decode_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > gpurun_out/plain_pf.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"xprep|wtile|prefill_gemm" -c 30 --csv --log-file gpurun_out/pf_launches.csv $PCMD > /dev/null 2>&1; echo ncu3_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wtile|prefill_gemm" -s 6 -c 2 -o gpurun_out/pf_full $PCMD > gpurun_out/pf_full.log 2>&1; echo ncu4_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
