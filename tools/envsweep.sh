# C3 (or $CFG) K-split under env settings: each arg is "NAME=V NAME=V"
for e in "$@"; do
  env $e timeout 300 python bench.py --config ${CFG:-C3} --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $BENCH_EXTRA > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "
import json
d=json.loads(open('gpurun_out/e.json').read().strip().splitlines()[-1])
print('$e |', d['config'].get('path'), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {n:round(x['ms'],4) for n,x in d.get('kernels',{}).items()}, {k:round(v,4) for k,v in d.get('step_ms',{}).items()})
" || tail -2 gpurun_out/e.err
done
