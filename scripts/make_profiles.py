"""Turn a round's ncu outputs (gpurun_out/) into the committed summaries under profiles/.

usage: python scripts/make_profiles.py r01 [workload_key]
  reads  gpurun_out/launches_<r>.csv   (ncu --metrics gpu__time_duration.sum launch list of bench.py)
         gpurun_out/decode_<r>.ncu-rep (ncu --set full of zq_kernel + decode_f8_kernel)
  writes profiles/<r>_launches.txt, profiles/<r>_ncu_full.txt, profiles/traffic.json[workload_key]
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]


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
        unit = d["Metric Unit"]
        v = float(d["Metric Value"]) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
        agg.setdefault(name, []).append(v)
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
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def prefill(r, key="c3_up_n8_b2048_g1"):
    """profiles/<r>_prefill_*.txt from gpurun_out/pf_launches.csv and pf_full.ncu-rep."""
    lp = os.path.join(ROOT, "gpurun_out", "pf_launches.csv")
    agg = launches(lp)
    tot = sum(sum(v) for v in agg.values())
    lines = ["# ncu launch list of `python bench.py --workload c3_up --steps 20 --warmup 3 --no-cpu-baseline --no-graph`",
             "# (--metrics gpu__time_duration.sum --clock-control none, kernels xprep|wtile|prefill_gemm; cold-cache,",
             "#  serialised -- compare shares)",
             f"{'kernel':60s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in agg.items():
        lines.append(f"{k:60s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v) / tot:7.3f}")
    open(os.path.join(ROOT, "profiles", f"{r}_prefill_launches.txt"), "w").write("\n".join(lines) + "\n")
    rep = os.path.join(ROOT, "gpurun_out", "pf_full.ncu-rep")
    out = ["# ncu --set full --clock-control none --import-source on: one launch each of wtile_kernel and",
           "# prefill_gemm_kernel (C3 up/gate 14336x4096, n=8, B=2048), from gpurun_out/pf_full.ncu-rep"]
    gemm_traffic = None
    for name, m in full(rep):
        out.append(name)
        for k, (v, u) in m.items():
            out.append(f"    {k:66s} {v} {u or ''}")
        if "prefill_gemm" in name:
            gemm_traffic = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    open(os.path.join(ROOT, "profiles", f"{r}_prefill_ncu_full.txt"), "w").write("\n".join(out) + "\n")
    if gemm_traffic is not None:
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        tj[key] = gemm_traffic
        json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines + out))


def main(r, key="c2_n16_b1_g1"):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{r}.csv")
    lines = [f"# ncu launch list (-k regex:'zq_kernel|decode_f8i') of `python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-graph`",
             "# (--metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised: PDL overlap",
             "#  of zq_kernel with decode_f8i_kernel is lost under ncu, so compare SHARES, not absolutes)",
             f"{'kernel':60s} {'launches':>8s} {'avg_us':>10s} {'total_us':>11s} {'share':>7s}"]
    agg = launches(lp)
    tot = sum(sum(v) for v in agg.values())
    steady = {k: v for k, v in agg.items()
              if not any(t in k for t in ("repack", "prep_factors", "inv_s", "factor_max", "factor_scale"))}
    tot_steady = sum(sum(v) for v in steady.values())
    for k, v in agg.items():
        lines.append(f"{k:60s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v):11.1f} {sum(v) / tot:7.3f}")
    lines.append("# per-call share (excluding one-off load_blocks kernels: repack / factor prep / inv_s):")
    for k, v in steady.items():
        lines.append(f"#   {k:56s} {sum(v) / tot_steady:6.3f}")
    open(os.path.join(ROOT, "profiles", f"{r}_launches.txt"), "w").write("\n".join(lines) + "\n")

    rep = os.path.join(ROOT, "gpurun_out", f"decode_{r}.ncu-rep")
    out = [f"# ncu --set full --clock-control none --import-source on, one launch of each kernel of the",
           "# decode pair (C2 4096x4096, n=16, k=16, bf16 factors, B=1), from gpurun_out/decode_" + r + ".ncu-rep"]
    traffic = 0.0
    for name, m in full(rep):
        out.append(name)
        for k, (v, u) in m.items():
            out.append(f"    {k:66s} {v} {u or ''}")
        traffic += to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    out.append(f"# pair DRAM traffic per call: {traffic:.0f} bytes")
    open(os.path.join(ROOT, "profiles", f"{r}_ncu_full.txt"), "w").write("\n".join(out) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj[key] = traffic
    tj["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per call of the roofline's dominant kernel, "
                   "from one ncu capture: decode keys = the zq_kernel + decode_f8i_kernel pair, "
                   "prefill (c3_*) keys = prefill_gemm_kernel; keys <workload>_n<n>_b<batch>_g<world>; "
                   "c4_b<batch>_g<world> = summed over the 256 launches of one C4 token-step "
                   "(scripts/gpu_c4_traffic.sh)")
    json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines + out))


def traffic_only(rep_name, key, regex):
    """profiles/traffic.json[key] = DRAM read + write bytes per call of the kernels matching
    `regex` in gpurun_out/<rep_name>.ncu-rep (one launch each)."""
    rep = os.path.join(ROOT, "gpurun_out", rep_name + ".ncu-rep")
    total, seen = 0.0, []
    for name, m in full(rep):
        if re.search(regex, name) and name not in seen:
            seen.append(name)
            total += to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj[key] = total
    json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    print(key, total, seen)


def c4_launches(r):
    """profiles/<r>_c4_launches.txt from gpurun_out/c4_launches.csv (scripts/gpu_sweeps.sh): the
    launches of one eager C4 token-step in order, zq then decode per group, 4 groups per layer."""
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", "c4_launches.csv"))))
    i = next(k for k, x in enumerate(rows) if x and x[0] == "ID")
    hdr = rows[i]
    us = []
    for x in rows[i + 1:]:
        d = dict(zip(hdr, x))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            us.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")) *
                       {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)))
    assert len(us) == 256, len(us)
    groups = ["{q,k,v}", "{o}", "{gate,up}", "{down}"]
    zq = {g: [] for g in groups}
    dec = {g: [] for g in groups}
    for j in range(128):
        g = groups[j % 4]
        (n0, t0), (n1, t1) = us[2 * j], us[2 * j + 1]
        assert "zq" in n0 and "decode" in n1
        zq[g].append(t0)
        dec[g].append(t1)
    tot = sum(t for _, t in us)
    lines = ["# ncu launch list of one eager C4 token-step (`python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph`)",
             "# (-k regex:'zq_mx|decode_mx', 128 launch pairs = 32 layers x 4 groups; --clock-control none,",
             "#  cold-cache and serialised: compare shares). Per group type, average over the layers:",
             f"{'group':14s} {'zq_us':>6s} {'decode_us':>10s} {'share':>7s}"]
    for g in groups:
        lines.append(f"{g:14s} {sum(zq[g]) / 32:6.2f} {sum(dec[g]) / 32:10.2f} {(sum(zq[g]) + sum(dec[g])) / tot:7.3f}")
    lines.append(f"# zq share of the token's kernel time: {sum(sum(v) for v in zq.values()) / tot:.3f}")
    open(os.path.join(ROOT, "profiles", f"{r}_c4_launches.txt"), "w").write("\n".join(lines) + "\n")


def traffic_csv(csv_path, key):
    """profiles/traffic.json[key] = DRAM read + write bytes summed over EVERY launch in an
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv` log (a whole step of
    many launches, e.g. one C4 token-step)."""
    import csv
    total, launches = 0.0, set()
    with open(csv_path) as f:
        rows = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(rows):
        if r.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += to_bytes(r["Metric Value"].replace(",", ""), r["Metric Unit"])
            launches.add(r["ID"])
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj[key] = total
    json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
    print(key, total, "bytes over", len(launches), "launches")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "prefill":
        prefill(sys.argv[1])
    elif len(sys.argv) > 1 and sys.argv[1] == "traffic":
        traffic_only(sys.argv[2], sys.argv[3], sys.argv[4])
    elif len(sys.argv) > 2 and sys.argv[2] == "c4":
        c4_launches(sys.argv[1])
    elif len(sys.argv) > 1 and sys.argv[1] == "traffic_csv":
        traffic_csv(sys.argv[2], sys.argv[3])
    else:
        main(*sys.argv[1:])
