set -x
O=gpurun_out/s5; mkdir -p $O
timeout 1200 python -m pytest tests/test_dist_gpu.py -m gpu -x -q -k "polymul_multi" > $O/multi.log 2>&1; echo "rc=$?" >> $O/multi.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "tests rc=$?" >> $O/gputest.log
