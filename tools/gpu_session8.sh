O=gpurun_out/s8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
for r in 1 2; do timeout 300 python tools/stage_times.py 32 128 5 >> $O/st.txt 2>&1; done
timeout 300 python tools/stage_times.py 28 128 5 >> $O/st28.txt 2>&1
