timeout 300 python -m pytest tests/test_cluster_gpu.py -x -q > gpurun_out/t_cluster.log 2>&1
for i in 1 2; do timeout 300 python bench.py --path cluster --config C1 --no-cpu-baseline --no-e2e --steps 200 --warmup 10 > gpurun_out/b_cl_$i.json 2>/dev/null; done
