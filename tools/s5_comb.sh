O=gpurun_out/s5l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
bash tools/c2_sweep2.sh > $O/sweep.log 2>&1; tail -8 $O/sweep.log
