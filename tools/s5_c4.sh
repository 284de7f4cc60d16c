O=gpurun_out/s5c
mkdir -p $O
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_parity_gpu.py tests/test_adi_gpu.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
for st in 1 2; do
  PSW_CLUSTER_ST=$st timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/c4_st$st.json 2> $O/c4_st$st.err
  python -c "
import json
d=json.loads([l for l in open('$O/c4_st$st.json') if l.startswith('{')][-1])
print('ST=$st', d['config'].get('path'), d['ms_per_step'], d['roofline']['frac'], d.get('step_ms'))
"
done
