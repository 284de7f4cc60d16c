timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --mode rows --config C3 --steps 3 --warmup 3 > gpurun_out/tr3.log 2>&1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/final_t3.log
