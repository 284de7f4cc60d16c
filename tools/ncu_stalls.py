"""Summarise an ncu report: per kernel duration, DRAM bytes, top stall reasons (pc samples)."""
import csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:70])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__grid_size", "launch__block_size"]:
        print("   ", k, d.get(k))
    vals = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                vals.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in vals) or 1
    print("    stalls:", ", ".join(f"{k} {100*v/tot:.0f}%" for v, k in sorted(vals, reverse=True)[:7]))
