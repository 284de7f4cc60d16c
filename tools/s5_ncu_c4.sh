O=gpurun_out/s5d
mkdir -p $O
timeout 300 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -s 1 -c 1 -o $O/prof_C4 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
tail -3 $O/ncu.log
