O=gpurun_out/s9; mkdir -p $O
for r in 1 2; do
timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_default.txt 2>&1
FPM_TOP4_THREADS=512 timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_t512.txt 2>&1
FPM_LIB=build/exp/q16k/libfpmul_b200.so timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_q16k.txt 2>&1
done
