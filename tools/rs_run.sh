timeout 600 python -m pytest tests/test_resweep_gpu.py -x -q > gpurun_out/t_resweep.log 2>&1
for c in C1 C3 C4; do timeout 300 python bench.py --path resweep --config $c --no-cpu-baseline --no-e2e --steps 20 --warmup 3 > gpurun_out/b_rs_$c.json 2>gpurun_out/b_rs_$c.err; done
