set -x
O=gpurun_out/s3; mkdir -p $O
FPM_L1_PIPE=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "basis_cvt or baseline_config" > $O/t2.log 2>&1; echo "rc=$?" >> $O/t2.log
for v in 0 2 0 2; do FPM_L1_PIPE=$v timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_$v.txt 2>&1; done
