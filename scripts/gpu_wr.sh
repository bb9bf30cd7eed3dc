#!/bin/bash
# A/B of the prefill W' restore: registers (mma.sync, default) vs tcgen05 + TMEM (BS_WRESTORE_TC=1)
O=gpurun_out/wr; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "prefill or full_size or smoke or numerics or dispatch or more_than" > $O/tests.log 2>&1; tail -3 $O/tests.log
for wl in c3_up c3_down; do
  timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline > $O/hm_$wl.json 2>/dev/null
  BS_WRESTORE_TC=1 timeout 300 python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu-baseline > $O/tc_$wl.json 2>/dev/null
  python scripts/bline.py < $O/hm_$wl.json; python scripts/bline.py < $O/tc_$wl.json
done
timeout 300 python bench.py --batch 48 --steps 200 --warmup 5 --no-cpu-baseline | python scripts/bline.py
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"absmax|xprep|wrestore|rgemv|prefill_gemm" -c 40 --csv --log-file $O/launches_c3_up.csv $PCMD > /dev/null 2>&1; echo ncu=$?
python scripts/launch_summary.py $O/launches_c3_up.csv 2>/dev/null | tail -6
