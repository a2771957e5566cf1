#!/bin/bash
# Build a variant of the library with extra defines on one source file (default k_decode):
#   tools/build_variant.sh NAME "-DFOO=1" [k_decode]
# -> variants/libqjl_NAME.so (git-ignored, travels to the GPU box); use with QJL_LIB=...
# The other objects come from paper_2406_03482_b200/csrc/build (run make first).
set -e
NAME=$1; DEFS=$2; SRCF=${3:-k_decode}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2406_03482_b200/csrc
OUT=$ROOT/variants/build_$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $DEFS"
nvcc $FLAGS -Xptxas -v -c $SRC/$SRCF.cu -o $OUT/$SRCF.o 2> $OUT/$SRCF.ptxas.log
OBJS=$(ls $SRC/build/*.o | grep -v "/$SRCF.o")
nvcc $ARCH -shared -cudart static -o $ROOT/variants/libqjl_$NAME.so $OUT/$SRCF.o $OBJS -Xlinker --exclude-libs,ALL
grep -A2 "k_udecodeILi8ELi2ELi4" $OUT/$SRCF.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo " -> variants/libqjl_$NAME.so"
rm -rf $OUT
