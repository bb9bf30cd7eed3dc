#!/bin/bash
# compute-sanitizer over every GPU path on small shapes (scripts/sanitize_case.py).
O=gpurun_out/r02
mkdir -p $O
python scripts/sanitize_case.py > $O/sanitize_plain.log 2>&1; echo plain=$?; tail -1 $O/sanitize_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > $O/sanitize_$tool.log 2>&1
  echo $tool=$?; tail -3 $O/sanitize_$tool.log
done
