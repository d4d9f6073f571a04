# Round-2 final evidence: full GPU suite, smoke, bench lines for configs 1-5 (+ reference arm at cfg5),
# cfg5 launch list, ncu --set full of the changed kernels.
set -x
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "tests rc=$?" >> $O/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 1 3 4 2; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv python tools/one_product.py 32 2 > $O/ncu_l.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg1.csv python tools/one_product.py 20 2 > $O/ncu_l1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_top8|fft_top4|l1_inner_rows" -c 4 -o $O/top4_l1 python tools/one_product.py 32 1 > $O/ncu_f.log 2>&1
ls -la $O
