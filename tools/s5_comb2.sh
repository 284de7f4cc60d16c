O=gpurun_out/s5m
mkdir -p $O
for sw in 1 0; do
PSW_COMBINE_SWEEP=$sw timeout 600 python bench.py --config C2 --P 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain$sw.log 2>&1 && \
PSW_COMBINE_SWEEP=$sw timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/l$sw.csv python bench.py --config C2 --P 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu$sw.log 2>&1
done
