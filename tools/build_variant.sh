#!/bin/bash
# Build a variant of the library with extra defines: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
# -> variants/libqjl_NAME.so (git-ignored, travels to the GPU box); use with QJL_LIB=...
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2406_03482_b200/csrc
OUT=$ROOT/variants/build_$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $DEFS"
pids=()
for f in api k_prefill k_scores k_decode_simt k_decode_tc k_decode_umma k_quant_tc k_qjlc k_orth; do
  nvcc $FLAGS -Xptxas -v -c $SRC/$f.cu -o $OUT/$f.o 2> $OUT/$f.ptxas.log &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p; done
nvcc $ARCH -shared -cudart static -o $ROOT/variants/libqjl_$NAME.so $OUT/*.o -Xlinker --exclude-libs,ALL
grep -A2 "k_udecodeILi8ELi2" $OUT/k_decode_umma.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo " -> variants/libqjl_$NAME.so"
rm -rf $OUT
