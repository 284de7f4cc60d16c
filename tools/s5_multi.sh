O=gpurun_out/s5g
mkdir -p $O
timeout 900 python -m pytest tests/test_fourier.py tests/test_prelim_gpu.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -25 $O/pytest.log
timeout 600 python tools/fourier_bench.py 4096 16 > $O/fourier.json 2> $O/fourier.err; cat $O/fourier.json; tail -3 $O/fourier.err
