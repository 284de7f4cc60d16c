O=gpurun_out/s5h
mkdir -p $O
for mr in 2048 1024 512; do
  for ck in 0; do
    PSW_HOST_MIN_ROW=$mr timeout 300 python tools/host_probe.py > $O/probe_$mr.json 2> $O/probe_$mr.err
    head -1 $O/probe_$mr.json
  done
done
tail -1 $O/probe_2048.json
