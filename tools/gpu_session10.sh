O=gpurun_out/s10; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
for c in 1 3; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg1.csv python tools/one_product.py 20 2 > $O/ncu1.log 2>&1
