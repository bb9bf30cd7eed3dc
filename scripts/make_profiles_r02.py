"""Round-2 evidence -> profiles/ (committed summaries).

usage: python scripts/make_profiles_r02.py
  reads  gpurun_out/r02/   (scripts/gpu_round2.sh, scripts/gpu_sanitize.sh)
         gpurun_out/rg/    (scripts/gpu_rg.sh: restore-and-multiply sweep + ncu)
  writes profiles/r02_*.json|txt and profiles/traffic.json keys
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R02 = os.path.join(ROOT, "gpurun_out", "r02")
RG = os.path.join(ROOT, "gpurun_out", "rg")
R02B = os.path.join(ROOT, "gpurun_out", "r02b")
PROF = os.path.join(ROOT, "profiles")
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def json_lines(path):
    out = []
    if not os.path.exists(path):
        return out
    for line in open(path):
        if line.startswith("{"):
            out.append(json.loads(line))
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    agg = OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        agg.setdefault((name, d.get("Grid Size", "")), []).append(v)
    return agg


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        res.append((re.sub(r"\(.*", "", d["Kernel Name"]), {k: (d.get(k), u.get(k)) for k in KEYS if k in d}))
    return res


def to_bytes(v, unit):
    return float(str(v).replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def write(name, text):
    with open(os.path.join(PROF, name), "w") as f:
        f.write(text if text.endswith("\n") else text + "\n")


def launch_summary(src, title, dst):
    if not os.path.exists(src):
        return
    agg = launches(src)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# {title}", "# (ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache and serialised,",
             "#  so PDL overlap is lost -- compare SHARES, not absolutes)",
             f"{'kernel':52s} {'grid':>14s} {'launches':>8s} {'avg_us':>9s} {'share':>6s}"]
    for (k, g), v in agg.items():
        lines.append(f"{k:52s} {g:>14s} {len(v):8d} {sum(v) / len(v):9.2f} {sum(v) / tot:6.3f}")
    write(dst, "\n".join(lines))


def ncu_summary(rep, title, dst, traffic_key=None, regex=None):
    if not os.path.exists(rep):
        return None
    out = [f"# {title}", f"# ncu --set full --clock-control none --import-source on ({os.path.relpath(rep, ROOT)})"]
    traffic = 0.0
    for name, m in full(rep):
        out.append(name)
        for k, (v, u) in m.items():
            out.append(f"    {k:66s} {v} {u or ''}")
        if regex is None or re.search(regex, name):
            traffic += to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    out.append(f"# DRAM read + write of the kernels above (one launch each): {traffic:.0f} bytes")
    write(dst, "\n".join(out))
    if traffic_key:
        tp = os.path.join(PROF, "traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        tj[traffic_key] = traffic
        json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    return traffic


def sweep_table(lines, title):
    out = [f"# {title}", f"{'workload':10s} {'B':>3s} {'kernel':>8s} {'us/call':>9s} {'GB/s alg':>9s} {'roofline':>9s} {'frac':>6s} {'clock':>6s}"]
    for d in lines:
        c = d["config"]
        r = d.get("roofline") or {}
        out.append(f"{c['workload'][:10]:10s} {c['batch']:3d} {r.get('kernel', '')[:8]:>8s} {d['ms_per_step'] * 1e3:9.2f} "
                   f"{d['value']:9.1f} {r.get('bound', ''):>9s} {r.get('frac', float('nan')):6.3f} "
                   f"{(d.get('clocks') or {}).get('sm_mhz', 0):6.0f}")
    return "\n".join(out)


def main():
    os.makedirs(PROF, exist_ok=True)
    # bench lines, verbatim
    for name in ["bench_c2_driver", "bench_c2", "bench_ref", "bench_c5", "bench_c4", "bench_c4_ungrouped", "bench_load",
                 "bench_compress", "bench_c3_up", "bench_c3_down", "bench_c2_b48"]:
        src = os.path.join(R02, name + ".json")
        ls = json_lines(src)
        if ls:
            write(f"r02_{name}.json", "\n".join(json.dumps(d) for d in ls))
    rb = json_lines(os.path.join(R02, "bench_rgemv_b8.jsonl"))
    if rb:
        write("r02_bench_rgemv_b8.json", "\n".join(json.dumps(d) for d in rb))
    # C5 per-rank shards
    sh = json_lines(os.path.join(R02, "shard_c5.jsonl"))
    if sh:
        out = ["# C5 (70B down_proj 8192 x 28672, n=12, B=1): rank 0's row shard of a G-way split timed alone on one",
               "# GPU (bench.py --workload c5 --shard G), V and s replicated; HBM floor = the shard's algorithmic bytes",
               "# at the measured copy bandwidth (BASELINE.md §3: G=8 floor 8.50 us)",
               f"{'G':>2s} {'rows':>5s} {'us/call':>9s} {'floor_us':>9s} {'frac':>6s}"]
        for d in sh:
            s = d["config"]["shard"]
            out.append(f"{s['of']:2d} {s['rows']:5d} {d['ms_per_step'] * 1e3:9.2f} {s['hbm_floor_us']:9.2f} {d['roofline']['frac']:6.3f}")
        write("r02_shard_c5.txt", "\n".join(out))
        write("r02_shard_c5.json", "\n".join(json.dumps(d) for d in sh))
    # batch sweeps: AUTO, and each path forced
    parts = []
    for fname, title in [("bsweep.jsonl", "AUTO path by batch (e4m3 decode B <= 5, restore-and-multiply 6..32, prefill above)"),
                         ("bsweep_decode.jsonl", "e4m3 decode forced (bench.py --kernel tc)"),
                         ("bsweep_rgemv.jsonl", "restore-and-multiply forced (bench.py --kernel rgemv)"),
                         ("bsweep_prefill.jsonl", "prefill forced (bench.py --kernel prefill)")]:
        ls = json_lines(os.path.join(R02, fname))
        if ls:
            parts.append(sweep_table(ls, title))
    if parts:
        write("r02_batch_sweep.txt", "\n\n".join(parts))
    # launch lists
    launch_summary(os.path.join(R02, "launches_c2.csv"),
                   "launch list of `python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph` (C2, B=1)",
                   "r02_launches_c2.txt")
    launch_summary(os.path.join(R02, "launches_c5.csv"),
                   "launch list of `python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-graph`",
                   "r02_launches_c5.txt")
    launch_summary(os.path.join(R02, "launches_c3_up.csv"),
                   "launch list of `python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph`",
                   "r02_launches_c3_up.txt")
    launch_summary(os.path.join(R02, "launches_c4.csv"),
                   "launch list of one eager C4 token-step (`bench.py --workload c4 --steps 1 --warmup 3 --no-graph`)",
                   "r02_launches_c4.txt")
    # ncu --set full
    ncu_summary(os.path.join(R02, "decode_c2.ncu-rep"), "C2 decode pair (zq_mx + decode_mx), one launch each",
                "r02_ncu_decode_c2.txt", "c2_n16_b1_g1")
    ncu_summary(os.path.join(R02, "decode_c5.ncu-rep"), "C5 decode pair (zq_mx + decode_mx), one launch each",
                "r02_ncu_decode_c5.txt", "c5_n12_b1_g1")
    ncu_summary(os.path.join(R02, "prefill_c3_up.ncu-rep"), "C3 up/gate prefill: W' restore (rgemv_kernel<16, true>) + GEMM, one launch each",
                "r02_ncu_prefill_c3_up.txt", "c3_up_n8_b2048_g1", regex="prefill_gemm")
    ncu_summary(os.path.join(R02, "rg_c5.ncu-rep"), "C5 restore-and-multiply (rgemv_kernel<16>, B=8, balanced ranges), one launch",
                "r02_ncu_rgemv_c5.txt", "c5_n12_b8_g1_rgemv", regex="rgemv")
    ncu_summary(os.path.join(R02, "rg_c2.ncu-rep"), "C2 restore-and-multiply (rgemv_kernel<16>, B=8), one launch",
                "r02_ncu_rgemv_c2.txt", "c2_n16_b8_g1_rgemv", regex="rgemv")
    # tests, smoke, sanitizer
    for src, dst in [("pytest_gpu.log", "r02_gpu_tests.txt"), ("smoke.log", "r02_smoke.txt")]:
        p = os.path.join(R02, src)
        if os.path.exists(p):
            lines = open(p).read().splitlines()
            write(dst, "\n".join(lines[-12:]))
    san = []
    for tool in ["plain", "memcheck", "racecheck", "synccheck", "initcheck"]:
        p = os.path.join(R02, f"sanitize_{tool}.log")
        if os.path.exists(p):
            lines = open(p).read().splitlines()
            san.append(f"## compute-sanitizer --tool {tool}" if tool != "plain" else "## plain run")
            san.extend(lines[-8:])
    if san:
        write("r02_sanitizer.txt", "# python scripts/sanitize_case.py (every GPU path, small shapes) under compute-sanitizer\n"
              + "\n".join(san))
    print("\n".join(sorted(f for f in os.listdir(PROF) if f.startswith("r02_"))))


if __name__ == "__main__":
    main()
