# Batch sweeps behind profiles/<r>_c4_batch_sweep.txt / <r>_c5_batch_sweep.txt, the C4 per-group
# launch list, and the DRAM-traffic captures (gpu_traffic.sh, gpu_c4_traffic.sh).
for b in 1 2 4 8 16; do
  printf "B=$b "; timeout 300 python bench.py --workload c4 --batch $b --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1
done > gpurun_out/c4_batch_sweep.txt
for b in 1 2 4 8 16 32 64; do
  printf "B=$b "; timeout 300 python bench.py --workload c5 --batch $b --steps 256 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
done > gpurun_out/c5_batch_sweep.txt
C4="python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $C4 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"zq_grouped|decode_f8i_grouped" -c 256 --csv --log-file gpurun_out/c4_launches.csv $C4 > /dev/null 2>&1; echo c4l_rc=$?
bash scripts/gpu_traffic.sh
bash scripts/gpu_c4_traffic.sh
