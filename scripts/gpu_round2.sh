#!/bin/bash
# Round-2 GPU evidence (one B200): full GPU tests + smoke, the bench lines of every workload
# (default C2 driver-style and long, reference arm, C5, C4 grouped / ungrouped, load, compress,
# prefill C3 up / down, C5 per-rank shards G = 2, 4, 8), the B = 1..16 sweeps, the ncu launch
# lists of the bench commands and --set full captures of the dominant kernels.
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvidia_smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c2_driver.json 2> $O/bench_c2_driver.err; echo b1=$?
timeout 600 python bench.py --sweep > $O/bench_c2.json 2> $O/bench_c2.err; echo b2=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo b3=$?
timeout 600 python bench.py --workload c5 --steps 2000 --warmup 20 > $O/bench_c5.json 2> $O/bench_c5.err; echo b4=$?
timeout 600 python bench.py --workload c4 --steps 200 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo b5=$?
timeout 600 python bench.py --workload c4 --steps 200 --warmup 5 --no-group --no-cpu-baseline > $O/bench_c4_ungrouped.json 2>/dev/null; echo b6=$?
timeout 600 python bench.py --workload load --steps 10 --warmup 3 > $O/bench_load.json 2> $O/bench_load.err; echo b7=$?
timeout 600 python bench.py --workload compress --steps 5 --warmup 2 > $O/bench_compress.json 2> $O/bench_compress.err; echo b8=$?
for wl in c3_up c3_down; do timeout 600 python bench.py --workload $wl --steps 300 --warmup 5 > $O/bench_$wl.json 2> $O/bench_$wl.err; echo pf=$?; done
for G in 2 4 8; do timeout 300 python bench.py --workload c5 --shard $G --steps 2000 --warmup 20 --no-cpu-baseline; done > $O/shard_c5.jsonl 2> $O/shard.err
for W in c2 c5; do for B in 1 2 3 4 5 6 8 12 16 24 32 48; do
  timeout 300 python bench.py --workload $W --batch $B --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep.jsonl 2> $O/bsweep.err
for W in c2 c5; do for B in 2 4 8 16; do
  timeout 300 python bench.py --workload $W --batch $B --kernel prefill --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep_prefill.jsonl 2>> $O/bsweep.err
for W in c2 c5; do for B in 1 3 8 16 32; do
  timeout 300 python bench.py --workload $W --batch $B --kernel rgemv --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep_rgemv.jsonl 2>> $O/bsweep.err
for W in c2 c5; do for B in 6 8 16; do
  timeout 300 python bench.py --workload $W --batch $B --kernel tc --steps 1000 --warmup 20 --no-cpu-baseline
done; done > $O/bsweep_decode.jsonl 2>> $O/bsweep.err
python scripts/bline.py < $O/bsweep.jsonl
# ncu: launch lists (cold-cache, serialised) and one --set full capture per dominant kernel,
# each after the same command exited 0 without ncu
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
timeout 300 $CMD > $O/plain_c2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_mx|decode_mx" -c 200 --csv --log-file $O/launches_c2.csv $CMD > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zq_mx|decode_mx" -s 40 -c 2 -o $O/decode_c2 $CMD > $O/ncu_c2.log 2>&1; echo ncu2=$?
CMD5="python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $CMD5 > $O/plain_c5.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_mx|decode_mx" -c 40 --csv --log-file $O/launches_c5.csv $CMD5 > /dev/null 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zq_mx|decode_mx" -s 10 -c 2 -o $O/decode_c5 $CMD5 > $O/ncu_c5.log 2>&1; echo ncu4=$?
PCMD="python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $PCMD > $O/plain_pf.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"absmax|xprep|wtile|prefill_gemm" -c 40 --csv --log-file $O/launches_c3_up.csv $PCMD > /dev/null 2>&1; echo ncu5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wtile|prefill_gemm" -s 6 -c 2 -o $O/prefill_c3_up $PCMD > $O/ncu_pf.log 2>&1; echo ncu6=$?
C4CMD="python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $C4CMD > $O/plain_c4.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq_mx|decode_mx" -c 256 --csv --log-file $O/launches_c4.csv $C4CMD > /dev/null 2>&1; echo ncu7=$?
RCMD="python bench.py --workload c2 --batch 8 --steps 20 --warmup 3 --no-cpu-baseline --no-graph"
timeout 300 $RCMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rgemv" -s 5 -c 1 -o $O/rg_c2 $RCMD > $O/ncu_rg.log 2>&1; echo ncu8=$?
echo done
