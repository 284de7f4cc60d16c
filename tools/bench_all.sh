# every BASELINE config through AUTO + the reference arm (round-end evidence)
for c in C0 C1 C4 C2 C3; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_auto_$c.json 2> gpurun_out/bench_auto_$c.err; done
timeout 600 python bench.py --config C3 --mode rows --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_auto_C3_rows1.json 2> gpurun_out/bench_auto_C3_rows1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
