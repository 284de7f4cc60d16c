O=gpurun_out/s5j
mkdir -p $O
timeout 300 python tools/l2_reuse_probe.py > $O/plain.log 2>&1 && \
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --csv --log-file $O/l2.csv python tools/l2_reuse_probe.py > $O/ncu.log 2>&1
tail -2 $O/plain.log
