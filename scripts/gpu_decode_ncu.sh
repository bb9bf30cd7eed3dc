# ncu evidence of the decode pair only (the decode part of gpu_round1.sh): launch list + --set full.
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_kernel|decode_f8i" -c 200 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_f8|zq_kernel" -s 40 -c 2 -o gpurun_out/decode_r01 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
