#!/bin/bash
O=gpurun_out/wr; mkdir -p $O
PCMD="python bench.py --workload c3_up --steps 3 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > /dev/null 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wrestore" -s 2 -c 1 -o $O/wr_c3 $PCMD > $O/ncu.log 2>&1; echo ncu=$?
