CMD="python bench.py --workload compress --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/cmp_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/cmp_launches.csv $CMD > gpurun_out/cmp_ncu.log 2>&1; echo rc=$?
