# prefill iteration: parity tests, bench lines for c3_up / c3_down, ncu launch list
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill" 2>&1 | tail -3
for wl in c3_up c3_down; do timeout 300 python bench.py --workload $wl --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/pf_$wl.json 2>gpurun_out/pf_$wl.err; echo rc=$?; tail -3 gpurun_out/pf_$wl.err; done
CMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 200 $CMD > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"xprep|wtile|prefill_gemm" -c 30 --csv --log-file gpurun_out/pf_launches.csv $CMD > /dev/null 2>&1; echo ncu=$?
if [ "$1" = "full" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wtile|prefill_gemm" -s 6 -c 2 -o gpurun_out/pf_full $CMD > gpurun_out/pf_full.log 2>&1; echo ncu_full=$?
fi
