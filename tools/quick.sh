# quick perf pass: AUTO on every config, kernels split, no CPU baseline / e2e
for c in ${CONFIGS:-C3 C1 C2 C4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $BENCH_EXTRA > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/q_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    k={n:round(v["ms"],4) for n,v in d.get("kernels",{}).items()}
    print(f, d["config"]["workload"], d["config"].get("path"), "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3), k)
PY
