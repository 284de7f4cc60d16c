# C2 (fp32, 65536 x 65536) over the partition counts of BASELINE configs[2]
for P in 8 16 32 64 128 256 512; do for pth in staged resweep; do timeout 600 python bench.py --config C2 --P $P --path $pth --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > gpurun_out/c2_${pth}_P$P.json 2>/dev/null; done; done
