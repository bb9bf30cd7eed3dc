#!/bin/bash
# C3 prefill evidence after the W' restore moved onto the restore-and-multiply pipeline:
# bench lines, the launch list and one ncu --set full capture of restore + GEMM.
set -u
O=gpurun_out/r02; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build_c3.log 2>&1 || { tail $O/build_c3.log; exit 1; }
for wl in c3_up c3_down; do timeout 600 python bench.py --workload $wl --steps 300 --warmup 5 > $O/bench_$wl.json 2> $O/bench_$wl.err; echo pf=$?; done
timeout 300 python bench.py --batch 48 --steps 300 --warmup 5 --no-cpu-baseline > $O/bench_c2_b48.json 2>/dev/null; echo b48=$?
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > $O/plain_pf.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"absmax|xprep|rgemv|prefill_gemm" -c 40 --csv --log-file $O/launches_c3_up.csv $PCMD > /dev/null 2>&1; echo ncu5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rgemv|prefill_gemm" -s 6 -c 2 -o $O/prefill_c3_up $PCMD > $O/ncu_pf.log 2>&1; echo ncu6=$?
for f in $O/bench_c3_up.json $O/bench_c3_down.json $O/bench_c2_b48.json; do python scripts/bline.py < $f; done
