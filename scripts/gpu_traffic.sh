# ncu --set full captures for the traffic figures of the C5 decode pair and the C3-down GEMM
C5="python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $C5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"decode_f8i|zq_kernel" -s 20 -c 2 -o gpurun_out/c5_full $C5 > gpurun_out/c5_full.log 2>&1; echo c5_rc=$?
D3="python bench.py --workload c3_down --steps 10 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $D3 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"prefill_gemm" -s 4 -c 1 -o gpurun_out/c3d_full $D3 > gpurun_out/c3d_full.log 2>&1; echo c3d_rc=$?
