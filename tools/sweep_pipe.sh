timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/s_t1.log
echo "C4 staged" >> gpurun_out/s_b1.log; timeout 200 python bench.py --config C4 --path staged --steps 20 --warmup 3 2>&1 | grep -E "^\{" >> gpurun_out/s_b1.log
