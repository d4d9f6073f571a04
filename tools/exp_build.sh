#!/bin/bash
# Experiment build of the CUDA library with extra nvcc defines, for A/B runs on the GPU box:
#   tools/exp_build.sh NAME -DFPM_X=1 ...   ->  build/exp/NAME/libfpmul_b200.so  (select with FPM_LIB=...)
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/exp/$NAME
mkdir -p $OUT/obj
NV="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $*"
make -s -C $ROOT/paper_1803_11301_b200/csrc -j8 OBJDIR=$OUT/obj OUT=$OUT/libfpmul_b200.so "NVFLAGS=$NV" $OUT/libfpmul_b200.so
rm -rf $OUT/obj  # (gpurun snapshots are capped at 512 MiB)
echo $OUT/libfpmul_b200.so
