export BITSTACK_LIB=$PWD/scripts/libbitstack_pref.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c2 or bf16 or grouped or split or zero or host or rank" > gpurun_out/pt_pref.log 2>&1; echo pref_rc=$?; tail -3 gpurun_out/pt_pref.log
for rep in 1 2; do
for v in def pref; do
  if [ $v = def ]; then unset BITSTACK_LIB; else export BITSTACK_LIB=$PWD/scripts/libbitstack_$v.so; fi
  for wl in c2 c5; do timeout 200 python bench.py --workload $wl --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/e_${v}_${wl}_$rep.json 2>/dev/null; done
  timeout 200 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/e_${v}_c4_$rep.json 2>/dev/null
done
done
python - <<'P'
import json
for v in ("def", "pref"):
    out = []
    for wl in ("c2", "c5", "c4"):
        for rep in (1, 2):
            try:
                d = json.loads(open(f"gpurun_out/e_{v}_{wl}_{rep}.json").read().strip().splitlines()[-1])
                out.append(f"{wl}#{rep} {d['ms_per_step']*1e3:.2f}")
            except Exception:
                out.append(f"{wl}#{rep} ERR")
    print(v, *out)
P
