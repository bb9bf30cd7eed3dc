#!/bin/bash
# Zq kernel iteration: numerics/parity tests, launch list of the C5 shard-8 pair, bench lines.
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "numerics or parity or fuzz or tp_gpu" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq|decode" -c 40 --csv --log-file gpurun_out/shard8_launch.csv python bench.py --workload c5 --shard 8 --steps 20 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zq|decode" -c 40 --csv --log-file gpurun_out/c2_launch.csv python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
for G in 1 8; do python bench.py --workload c5 --shard $G --steps 2000 --warmup 50 --no-cpu-baseline; done > gpurun_out/shard.jsonl 2>&1
python bench.py --steps 5000 --warmup 50 --no-cpu-baseline >> gpurun_out/shard.jsonl 2>&1
python bench.py --steps 5000 --warmup 50 --no-cpu-baseline --batch 8 >> gpurun_out/shard.jsonl 2>&1
python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/shard.jsonl 2>&1
python scripts/bline.py < gpurun_out/shard.jsonl
