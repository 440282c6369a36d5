#!/bin/bash
# Build a kernel variant of libndconv_b200.so with extra nvcc defines into tools/variants/.
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR"
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
S=$ROOT/paper_1711_11224_b200/csrc; O=/tmp/variant_$NAME; rm -rf $O; mkdir -p $O $ROOT/tools/variants
SRCS=$(cd $ROOT && python -c "from paper_1711_11224_b200.build import SOURCES; print(' '.join(s[:-3] for s in SOURCES))")
N=$(echo $SRCS | wc -w)
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden $DEFS \
       -I $ROOT/include -c $S/$f.cu -o $O/$f.o &
done; wait
[ $(ls $O/*.o | wc -l) -eq $N ] || { echo "variant $NAME: compile failed" >&2; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/tools/variants/lib_$NAME.so $O/*.o \
     -Xlinker --version-script=$S/exports.map -ldl -lpthread
echo $ROOT/tools/variants/lib_$NAME.so
