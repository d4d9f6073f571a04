# round-2 session 2: small-config bench lines, cfg1 launch list, ncu full captures of the FFT kernels
set -x
O=gpurun_out/s2; mkdir -p $O
for c in 1 3 4 2; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg1.csv python tools/one_product.py 20 2 > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_tile_tower -c 1 -o $O/tower12 python tools/one_product.py 32 1 > $O/ncu_tower.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_top4 -c 2 -o $O/top4 python tools/one_product.py 32 1 > $O/ncu_top4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"carry_rows|conv_rows|conv256_a_encode|decode_conv_a" -c 4 -o $O/conv python tools/one_product.py 32 1 > $O/ncu_conv.log 2>&1
ls -la $O
