O=gpurun_out/s5k
mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_prelim_gpu.py tests/test_fourier.py -m gpu -q -x -p no:cacheprovider -k "not large and not default" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
tail -15 $O/memcheck.log
