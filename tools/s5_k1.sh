O=gpurun_out/s5i
mkdir -p $O
timeout 1200 python -m pytest tests/test_resweep_gpu.py tests/test_parity_gpu.py tests/test_sharded_gpu.py tests/test_properties_gpu.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
for c in C2 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/$c.json 2> $O/$c.err
  python -c "
import json
d=json.loads([l for l in open('$O/$c.json') if l.startswith('{')][-1])
print('$c', d['config'].get('path'), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), {k:round(v['ms'],4) for k,v in d['kernels'].items()})
"
done
