# C2 (fp32, 65536 x 65536) over the partition counts of BASELINE configs[2], AUTO path
O=gpurun_out/c2sweep
mkdir -p $O
for P in 8 16 32 64 128 256 512; do
  timeout 600 python bench.py --config C2 --P $P --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/P$P.json 2> $O/P$P.err
done
python - <<'PY'
import json,glob
out=[]
for P in (8,16,32,64,128,256,512):
    try:
        d=json.loads([l for l in open(f"gpurun_out/c2sweep/P{P}.json") if l.startswith("{")][-1])
    except Exception as e:
        out.append(f"P={P} ERR {e}"); continue
    k={n:round(v["ms"],3) for n,v in d.get("kernels",{}).items()}
    out.append(f"C2 fp32 65536x65536 P={P:<4d} {d['config'].get('path'):8s} {d['ms_per_step']:7.3f} ms  {d['value']:.3g} unknowns/s  HBM frac {d['roofline']['frac']:.3f}  kernels {k}")
open("gpurun_out/c2sweep/summary.txt","w").write("\n".join(out)+"\n")
print("\n".join(out))
PY
