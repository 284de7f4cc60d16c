O=gpurun_out/s5n
mkdir -p $O
timeout 600 python -m pytest tests/test_threads_gpu.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -8 $O/pytest.log
