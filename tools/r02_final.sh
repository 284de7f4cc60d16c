# round-2 final evidence pass: tests, smoke, default bench (C3), reference arm,
# the other configs, ncu launch lists (C3, C2, C1) + full captures (C3 K1/K3, C1)
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in C0 C1 C2 C4 C4c; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python tools/adi_bench.py > $O/adi.json 2>&1
timeout 600 python tools/fourier_bench.py 4096 16 > $O/fourier.json 2>&1
timeout 120 python tools/readpeak.py > $O/readpeak.json 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu_launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_l3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu_launches_C2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_l2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/ncu_launches_C1.csv python bench.py --config C1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_l1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_part_tma|rs_solve_tma_st" -s 2 -c 2 -o $O/prof_C3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_C3.log 2>&1
timeout 600 python tools/setup_bench.py > $O/setup_bench.json 2> $O/setup_bench.txt
timeout 600 python tools/adi_parts.py > $O/adi_parts.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -s 1 -c 1 -o $O/prof_C4 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_C4.log 2>&1
