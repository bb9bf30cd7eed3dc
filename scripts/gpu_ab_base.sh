# same-box A/B: base (HEAD), pf (+U' prefetch), def (current tree: P-generalised, R4 P1), p2
for rep in 1 2; do
for v in base pf def p2; do
  if [ $v = def ]; then unset BITSTACK_LIB; else export BITSTACK_LIB=$PWD/scripts/libbitstack_$v.so; fi
  for wl in c2 c5; do timeout 300 python bench.py --workload $wl --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/ab2_${v}_${wl}_$rep.json 2>/dev/null; done
done
done
python - <<'P'
import json
for v in ("base", "pf", "def", "p2"):
    out = []
    for wl in ("c2", "c5"):
        for rep in (1, 2):
            f = f"gpurun_out/ab2_{v}_{wl}_{rep}.json"
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1])
                out.append(f"{wl}#{rep} {d['ms_per_step']*1e3:.2f}us")
            except Exception as e:
                out.append(f"{wl}#{rep} ERR")
    print(v, *out)
P
