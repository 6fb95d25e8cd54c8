"""Digest an ncu report into small text (run next to the report; the .ncu-rep files are
tens of MB and do not fit gpurun's return budget).

    python scripts/ncu_digest.py <rep.ncu-rep> <out.txt> [top_n]

Writes the details page (speed of light, occupancy, warp-state and pipe metrics) and the
top SASS instructions by warp-stall samples with their opcode mix totals.
"""
import collections
import csv
import subprocess
import sys


def main(rep, out, top=60):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    raw_keep = {}
    if len(rr) >= 3:
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg",
                  "sm__cycles_elapsed.avg", "lts__t_sector_hit_rate.pct"):
            if k in rr[0]:
                raw_keep[k] = (rr[-1][rr[0].index(k)], rr[1][rr[0].index(k)])
    rows = list(csv.reader(src.splitlines()))
    hdr = None
    data = []
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    stall_key = "Warp Stall Sampling (All Samples)"
    for d in data:
        try:
            d["_s"] = int(d.get(stall_key, "0") or 0)
            d["_e"] = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            d["_s"], d["_e"] = 0, 0
    tot_s = sum(d["_s"] for d in data) or 1
    tot_e = sum(d["_e"] for d in data) or 1
    ops = collections.Counter()
    ops_s = collections.Counter()
    for d in data:
        toks = d["Source"].strip().split(" ")
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        parts = op.split(".")
        op = ".".join(parts[:2]) if parts[0] == "IMAD" else parts[0]     # IMAD.WIDE / .IADD / .MOV / .HI
        ops[op] += d["_e"]
        ops_s[op] += d["_s"]
    with open(out, "w") as f:
        f.write(det)
        f.write("\n=== raw metrics ===\n")
        for k, (v, unit) in raw_keep.items():
            f.write(f"{k}    {v} {unit}\n")
        f.write("\n=== SASS opcode mix (executed warp instructions, share of stall samples) ===\n")
        for op, e in ops.most_common(25):
            f.write(f"{op:12s} exec {100 * e / tot_e:5.1f}%  stalls {100 * ops_s[op] / tot_s:5.1f}%\n")
        # per-reason stall columns of the source page (when the SourceCounters section has them)
        reasons = [k for k in (hdr or []) if k.lower().startswith("stall_") or k.startswith("Warp Stall Sampling (")]
        f.write("\n=== source-page columns ===\n" + " | ".join(hdr or []) + "\n")
        def num(d, k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        if reasons:
            f.write("\n=== stall reasons over the kernel (share of samples) ===\n")
            tot = {k: sum(num(d, k) for d in data) for k in reasons}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
                f.write(f"{k:50s} {100 * v / tot_s:6.2f}%\n")
        # code regions delimited by barriers: where the samples sit (load / pass / exchange phases)
        f.write("\n=== regions between barriers (instruction index range, executed share, stall share, top reasons) ===\n")
        start = 0
        def flush(a, b, label):
            seg = data[a:b]
            if not seg:
                return
            e = sum(d["_e"] for d in seg)
            st = sum(d["_s"] for d in seg)
            top3 = ""
            if reasons:
                rs = sorted(((sum(num(d, k) for d in seg), k) for k in reasons if not k.endswith("(All Samples)")), reverse=True)[:3]
                top3 = ", ".join(f"{k.replace('stall_', '')} {100 * v / max(st, 1):.0f}%" for v, k in rs)
            mem = sum(1 for d in seg if any(t in d["Source"] for t in ("LDG", "STG")))
            f.write(f"[{a:5d},{b:5d}) exec {100 * e / tot_e:5.1f}%  stalls {100 * st / tot_s:5.1f}%  ldg/stg {mem:3d}  {label}  {top3}\n")
        for idx, d in enumerate(data):
            if "BAR" in d["Source"] or "EXIT" in d["Source"]:
                flush(start, idx + 1, d["Source"].strip()[:28])
                start = idx + 1
        flush(start, len(data), "end")
        f.write(f"\n=== top {top} SASS lines by stall samples (of {tot_s}) ===\n")
        for d in sorted(data, key=lambda d: -d["_s"])[:top]:
            f.write(f"{100 * d['_s'] / tot_s:5.2f}%  exec {d['_e']:>10d}  {d['Address'][-5:]}  {d['Source'].strip()[:90]}\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 60)
