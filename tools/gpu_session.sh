set -x
mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s1/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/s1/gputest.log
timeout 600 python bench.py > gpurun_out/s1/bench5.json 2> gpurun_out/s1/bench5.err; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/s1/launches.csv python tools/one_product.py > gpurun_out/s1/ncu.log 2>&1; echo ncu rc=$?
