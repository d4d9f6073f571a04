# A/B stage times: bash tools/gpu_ab.sh OUTDIR VARIANT...  (VARIANT = build/exp/NAME or "default")
O=$1; shift; mkdir -p $O
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_default.txt 2>&1
  else FPM_LIB=$v/libfpmul_b200.so timeout 300 python tools/stage_times.py 32 128 5 >> $O/st_$(basename $v).txt 2>&1; fi
done; done
