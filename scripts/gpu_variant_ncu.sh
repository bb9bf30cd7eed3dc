#!/bin/bash
# ncu --set full of the decode pair for each decode variant (C2, B=1): the pipe / DRAM / issue
# utilisation behind DESIGN.md §6.2's variant table
O=gpurun_out/r02v
mkdir -p $O
LIB=paper_2410_23918_b200/libbitstack.so
cp $LIB /tmp/lib_orig.so
CMD="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph"
for v in ${VARS:-base r2s4 occ2 skel}; do
  cp scripts/variants/lib_$v.so $LIB
  timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:"decode_mx" -s 40 -c 1 -o $O/dec_$v $CMD > $O/ncu_$v.log 2>&1; echo $v=$?
done
cp /tmp/lib_orig.so $LIB
