"""Copy a round's GPU evidence (gpurun_out/rNN) into profiles/: bench lines,
the ncu launch list, per-kernel DRAM traffic of one solve
(profiles/ncu_traffic.json, read by bench.py's roofline.traffic), the
`--set full` details pages and stall summaries.

    python tools/make_profiles.py r02
"""
import csv
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", rnd)
rnd = sys.argv[2] if len(sys.argv) > 2 else rnd  # output prefix
dst = os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    out = {}
    for r in rows[1:]:
        k = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
        out.setdefault(k, {})[r[ix["Metric Name"]]] = v * scale
    return out


for f in glob.glob(os.path.join(src, "bench_*.json")) + glob.glob(os.path.join(src, "*.json")):
    if os.path.getsize(f):
        shutil.copy(f, os.path.join(dst, f"{rnd}_" + os.path.basename(f)))

traffic_path = os.path.join(dst, "ncu_traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for f in glob.glob(os.path.join(src, "ncu_launches_*.csv")):
    cfg = os.path.basename(f)[len("ncu_launches_"):-4]
    shutil.copy(f, os.path.join(dst, f"{rnd}_" + os.path.basename(f)))
    L = launches(f)
    ids = sorted(L)
    # one solve = the kernels between two rs_part launches (skip fills / flushes)
    names = [n for _, n in ids]
    solve_kernels = [k for k in ids if not any(x in k[1] for x in ("fill_", "flush", "l2_"))]
    starts = [i for i, k in enumerate(solve_kernels) if "part" in k[1] or "cluster" in k[1] or "fused" in k[1]]
    if not starts:
        continue
    a = starts[-1]
    one = solve_kernels[a:a + (starts[1] - starts[0] if len(starts) > 1 else len(solve_kernels) - a)]
    rd = sum(L[k].get("dram__bytes_read.sum", 0) for k in one)
    wr = sum(L[k].get("dram__bytes_write.sum", 0) for k in one)
    per = [{"kernel": k[1].split("(")[0][-60:], "ms": L[k].get("gpu__time_duration.sum", 0) * 1e3,
            "dram_read": L[k].get("dram__bytes_read.sum", 0),
            "dram_write": L[k].get("dram__bytes_write.sum", 0)} for k in one]
    path = ("resweep" if any("rs_part" in k[1] for k in one) else
            "cluster" if any("cluster" in k[1] for k in one) else
            "fused" if any("fused" in k[1] for k in one) else "other")
    traffic[f"{cfg}:{path}"] = {"dram_bytes_per_solve": rd + wr, "dram_read": rd, "dram_write": wr,
                                "kernels": per, "source": f"profiles/{rnd}_ncu_launches_{cfg}.csv"}
json.dump(traffic, open(traffic_path, "w"), indent=1)

with open(os.path.join(dst, f"{rnd}_ncu_stalls.txt"), "w") as out:
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        base = os.path.basename(rep)[:-8]
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                             text=True).stdout
        open(os.path.join(dst, f"{rnd}_{base}_details.csv"), "w").write(det)
        s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), rep],
                           capture_output=True, text=True).stdout
        out.write(f"== {base}\n{s}\n")
print(json.dumps(traffic, indent=1)[:1500])
