"""Summarise ncu outputs into profiles/ text files (run here, no GPU needed).

    python scripts/summarize_ncu.py <launches.csv> <out_prefix> [rep.ncu-rep ...]
"""
import collections
import csv
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"source: {path}\n(cold-cache, serialised launches: compare SHARES, not absolutes)\n")
        for k, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k:40s} launches {c:5d}  total {ns / 1e3:10.1f} us  avg {ns / c / 1e3:8.2f} us  share {100 * ns / tot:5.1f}%\n")
    print(open(out).read())


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Instructions"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]


def report(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    lines = []
    kname = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in KEYS:
            lines.append(f"{d['Metric Name']:40s} {d.get('Metric Value', ''):>16s} {d.get('Metric Unit', '')}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    stalls = []
    for name, unit, val in zip(h, u, v):
        if name in RAW:
            lines.append(f"{name:60s} {val:>16s} {unit}")
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls.append((float(val.replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    lines.append("warp stall samples (share): " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    with open(out, "w") as f:
        f.write(f"ncu --set full --clock-control none: {kname}\n")
        f.write("\n".join(lines) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] != "/dev/null":
        launches(sys.argv[1], sys.argv[2] + "_launches.txt")
    for rep in sys.argv[3:]:
        tag = rep.split("/")[-1].replace(".ncu-rep", "")
        report(rep, f"{sys.argv[2]}_{tag}.txt")
