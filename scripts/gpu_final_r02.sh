#!/bin/bash
# Round-end verification on a fresh box: build, smoke, the default bench line, the reference arm.
set -u
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
tail -2 $O/smoke.log; python scripts/bline.py < $O/bench_default.json; python scripts/bline.py < $O/bench_reference.json
