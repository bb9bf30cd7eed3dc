# Ring-depth A/B of decode_f8i (libraries from paper_2410_23918_b200/build.py with
# -DBS_F8_STAGES=<cap> [-DBS_F8_SMEM_KB=<kb>]): us per call (C2, C5, C2 at batch 2 / 4) and
# ms per token (C4).  Usage: bash scripts/exp_stages.sh "base st8 st6"
for rep in 1 2; do
for v in ${1:-base st8}; do
  if [ "$v" = "base" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_$v.so"; fi
  for w in c2 c5 c4 c2b2 c2b4; do
    st=2000; a=""; ww=$w
    [ $w = c4 ] && st=200
    [ $w = c2b2 ] && { ww=c2; a="--batch 2"; }
    [ $w = c2b4 ] && { ww=c2; a="--batch 4"; }
    env $L timeout 300 python bench.py --workload $ww $a --steps $st --warmup 20 --no-cpu-baseline > gpurun_out/st_${v}_$w.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/st_${v}_$w.json').read().strip().splitlines()[-1]); print('$rep $v $w', '%.2f' % (d['ms_per_step']*1e3))"
  done
done
done
