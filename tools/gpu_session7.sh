set -x
O=gpurun_out/s7; mkdir -p $O
timeout 1500 python -m pytest tests/test_dist_gpu.py tests/test_dist_ipc.py -m gpu -x -q > $O/dist.log 2>&1; echo "rc=$?" >> $O/dist.log
