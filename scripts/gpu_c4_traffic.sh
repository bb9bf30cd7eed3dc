# DRAM bytes of one C4 token-step (the 128 grouped zq_mx + decode_mx pairs, eager launches):
# skip the 3 warm-up token-steps and the launch-counting one, capture the next token-step.
C4="python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-graph"
timeout 600 $C4 > gpurun_out/c4_plain.json 2> gpurun_out/c4_plain.err; echo plain_rc=$?
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"zq_mx_grouped|decode_mx_grouped" -s 1024 -c 256 --csv --log-file gpurun_out/c4_dram.csv \
  $C4 > gpurun_out/c4_ncu.log 2>&1; echo ncu_rc=$?
python scripts/make_profiles.py traffic_csv gpurun_out/c4_dram.csv c4_b1_g1
