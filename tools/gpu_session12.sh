O=gpurun_out/s12; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
for r in 1 2; do
timeout 300 python tools/stage_times.py 32 64 5 >> $O/st64_default.txt 2>&1
FPM_LIB=build/exp/q64k16/libfpmul_b200.so timeout 300 python tools/stage_times.py 32 64 5 >> $O/st64_q16.txt 2>&1
done
