O=gpurun_out/s11; mkdir -p $O
FPM_LIB=build/exp/poly2/libfpmul_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "baseline_config" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
bash tools/gpu_ab.sh $O default build/exp/poly2
