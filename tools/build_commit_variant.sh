#!/bin/bash
# Build libndconv_b200.so from the sources of an earlier commit into tools/variants/ (A/B of
# kernel changes with tools/ab_kbench.sh).  usage: tools/build_commit_variant.sh COMMIT NAME
set -e
C=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/commit_$NAME; rm -rf $T; mkdir -p $T
git -C $ROOT archive $C paper_1711_11224_b200/csrc include | tar -x -C $T
S=$T/paper_1711_11224_b200/csrc; O=$T/obj; mkdir -p $O $ROOT/tools/variants
SRCS=$(cd $S && ls ndc_*.cu)
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
       -I $T/include -c $S/$f -o $O/${f%.cu}.o &
done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/tools/variants/lib_$NAME.so $O/*.o \
     -Xlinker --version-script=$S/exports.map -ldl -lpthread
echo $ROOT/tools/variants/lib_$NAME.so
