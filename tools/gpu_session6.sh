set -x
O=gpurun_out/s6; mkdir -p $O
timeout 600 python tools/multi_product.py 32 8 2 > $O/multi8.log 2>&1
FPM_SHARD_CVT=0 timeout 600 python tools/multi_product.py 32 8 2 > $O/multi8_noshard.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file $O/launches_p8.csv python tools/multi_product.py 32 8 1 > $O/ncu_p8.log 2>&1
