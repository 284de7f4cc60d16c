O=gpurun_out/s5e
mkdir -p $O
timeout 600 python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"rs_part_tma|rs_solve_tma_st" -s 2 -c 2 -o $O/prof_C2 python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
tail -3 $O/ncu.log | cut -c1-300
