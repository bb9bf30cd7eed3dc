# Decode skeleton timing (wrong results, timing only): libraries built from decode_f8i.cuh with
# -DBS_EXP_SKEL (no expansion / TMEM stores / MMAs), -DBS_EXP_NOSIGN (no sign-tile copies), both.
for v in base skel nosign skelns; do
  if [ "$v" = "base" ]; then L=""; else L="BITSTACK_LIB=scripts/libbitstack_$v.so"; fi
  for w in c2 c5; do
    env $L timeout 300 python bench.py --workload $w --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/sk_${v}_$w.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sk_${v}_$w.json')); print('$v $w', 'us %.2f' % (d['ms_per_step']*1e3))"
  done
done
