#!/bin/bash
O=gpurun_out/wr; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "prefill or more_than or smoke" > $O/tests2.log 2>&1; tail -2 $O/tests2.log
for wl in c3_up c3_down; do
  timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | python scripts/bline.py
  BS_WRESTORE_TC=1 timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | python scripts/bline.py
done
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"wrestore" -c 3 $PCMD 2>&1 | grep -E "duration|issue_active|inst_executed" | tail -3
