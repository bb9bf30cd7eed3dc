"""Summarise an ncu report: SOL, pipes, DRAM bytes, stall reasons per barrier/instruction."""
import csv, io, re, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2]))

def main(rep):
    d = raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "launch__registers_per_thread"]
    for k in keys:
        for kk, v in d.items():
            if kk == k:
                print(f"{k:70s} {v}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
    tot = sum(float(x["Warp Stall Sampling (All Samples)"] or 0) for x in data)
    agg = {}
    for i, x in enumerate(data):
        m = re.search(r"TRYWAIT P\d, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", x["Source"])
        if m:
            s = sum(float(data[j]["Warp Stall Sampling (All Samples)"] or 0) for j in range(i, min(i + 2, len(data))))
            agg[m.group(1)] = agg.get(m.group(1), 0) + s
    print("total stall samples", tot)
    print("barrier waits (smem offset: samples):", {k: int(v) for k, v in sorted(agg.items())})
    top = sorted(data, key=lambda x: -float(x["Warp Stall Sampling (All Samples)"] or 0))[:12]
    for x in top:
        print(x["Address"][-5:], x["Warp Stall Sampling (All Samples)"].rjust(6), x["Source"][:90])

if __name__ == "__main__":
    main(sys.argv[1])


def regions(rep):
    """Stall samples per warp-role code region (markers: first UBLKCP/UTCHMMA/F2FP/STTM/ERRBAR)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
    marks = {}
    for i, x in enumerate(data):
        for key in ("UBLKCP", "UTCHMMA", "F2FP", "STTM", "LDTM", "ERRBAR"):
            if key in x["Source"] and key not in marks:
                marks[key] = i
    order = sorted(marks.items(), key=lambda kv: kv[1])
    print("markers:", order)
    bounds = [0] + [i for _, i in order] + [len(data)]
    names = ["setup"] + [k for k, _ in order]
    for nm, a, b in zip(names, bounds, bounds[1:]):
        s = sum(float(x["Warp Stall Sampling (All Samples)"] or 0) for x in data[a:b])
        inst = sum(float(x["Instructions Executed"] or 0) for x in data[a:b])
        print(f"  region from {nm:8s}: samples {s:7.0f}  warp-inst executed {inst:10.0f}")
