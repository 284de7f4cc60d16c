timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/cb_t1.log
for c in C1 C4; do echo "$c staged" >> gpurun_out/cb_b1.log; timeout 100 python bench.py --config $c --path staged --steps 50 --warmup 5 2>&1 | grep -E "^\{" >> gpurun_out/cb_b1.log; done
