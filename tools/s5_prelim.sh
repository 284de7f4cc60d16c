O=gpurun_out/s5b
mkdir -p $O
timeout 900 python -m pytest tests/test_prelim_gpu.py -m gpu -q -x -s -p no:cacheprovider > $O/pytest_prelim.log 2>&1; echo "rc=$?" >> $O/pytest_prelim.log
tail -30 $O/pytest_prelim.log
timeout 600 python tools/setup_bench.py > $O/setup_bench.json 2> $O/setup_bench.err
cat $O/setup_bench.json; grep "psw setup" $O/setup_bench.err
