timeout 600 python -m pytest tests/test_resweep_gpu.py -x -q > gpurun_out/t_resweep.log 2>&1
for pth in staged resweep; do timeout 300 python bench.py --path $pth --config C4 --no-cpu-baseline --no-e2e --steps 50 --warmup 5 > gpurun_out/b_c4_$pth.json 2>gpurun_out/b_c4_$pth.err; done
