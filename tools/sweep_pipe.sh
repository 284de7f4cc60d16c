set -x
python bench.py > gpurun_out/r01_bench_C1.json 2> gpurun_out/r01_bench_C1.err
for c in C0 C4; do python bench.py --config $c > gpurun_out/r01_bench_$c.json 2> gpurun_out/r01_bench_$c.err; done
python bench.py --config C2 --steps 5 --warmup 3 > gpurun_out/r01_bench_C2.json 2> gpurun_out/r01_bench_C2.err
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r01_bench_C3.json 2> gpurun_out/r01_bench_C3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01_bench_reference.json 2> gpurun_out/r01_bench_reference.err
python bench.py --mode rows --config C3 --steps 5 --warmup 3 > gpurun_out/r01_bench_C3_rows1.json 2> gpurun_out/r01_bench_C3_rows1.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_ncu_launches_C1.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_r_kernel -s 2 -c 1 -o gpurun_out/r01_fused_C1 python bench.py --steps 2 --warmup 2 > gpurun_out/ncu_full_c1.log 2>&1
ncu --set full --clock-control none -k regex:"fwd_s_kernel|bwd_s_kernel" -s 2 -c 2 -o gpurun_out/r01_staged_S_C4 python bench.py --config C4 --steps 2 --warmup 2 > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --clock-control none -k regex:"fwd_r_kernel|bwd_r_kernel" -s 2 -c 2 -o gpurun_out/r01_staged_R_C3 python bench.py --config C3 --steps 1 --warmup 1 > gpurun_out/ncu_full_c3.log 2>&1
