#!/bin/bash
# full GPU tests, then the C3 / rgemv evidence after the out-of-line W' row bound
O=gpurun_out/r02; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo tests=$?; tail -2 $O/pytest_gpu.log
for wl in c3_up c3_down; do timeout 600 python bench.py --workload $wl --steps 300 --warmup 5 > $O/bench_$wl.json 2> $O/bench_$wl.err; python scripts/bline.py < $O/bench_$wl.json; done
timeout 300 python bench.py --batch 48 --steps 300 --warmup 5 --no-cpu-baseline > $O/bench_c2_b48.json 2>/dev/null; python scripts/bline.py < $O/bench_c2_b48.json
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline | python scripts/bline.py
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > $O/plain_pf.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"absmax|xprep|rgemv|prefill_gemm" -c 40 --csv --log-file $O/launches_c3_up.csv $PCMD > /dev/null 2>&1; echo ncu5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rgemv|prefill_gemm" -s 6 -c 2 -o $O/prefill_c3_up $PCMD > $O/ncu_pf.log 2>&1; echo ncu6=$?
