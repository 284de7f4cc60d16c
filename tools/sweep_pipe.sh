PSW_FUSED_LAG=3 timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "fused or golden" 2>&1 | tail -3 > gpurun_out/lt_b1.log
for L in 3 0; do echo "C1 fused LAG=$L" >> gpurun_out/lt_b1.log; PSW_FUSED_VERBOSE=1 PSW_FUSED_LAG=$L timeout 100 python bench.py --config C1 --path fused --steps 50 --warmup 5 2>&1 | grep -E "^\{|fused:" | sort -u | head -2 >> gpurun_out/lt_b1.log; done
PSW_FUSED_LAG=3 timeout 100 python tools/trace_fused.py >> gpurun_out/lt_b1.log 2>&1
