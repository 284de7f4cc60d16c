cd _old
for c in C3 C2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/old_$c.json 2> ../gpurun_out/old_$c.err; done
cd ..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rs_part|rs_solve" -s 2 -c 2 -o gpurun_out/prof_C3_rs python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rs.log 2>&1
