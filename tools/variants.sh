# C3 (or $CFG) across library variants: VARIANTS="default rs4 ..."
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset PSW_LIB_VARIANT; else export PSW_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --config ${CFG:-C3} --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $BENCH_EXTRA > gpurun_out/v_${CFG:-C3}_$v.json 2> gpurun_out/v_${CFG:-C3}_$v.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/v_${CFG:-C3}_$v.json').read().strip().splitlines()[-1])
print('$v', d['config'].get('path'), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {n:round(x['ms'],4) for n,x in d.get('kernels',{}).items()})
" || tail -3 gpurun_out/v_${CFG:-C3}_$v.err
done
