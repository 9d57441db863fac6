#!/bin/bash
# Build a librtssph.so variant for A/B runs (scripts/ab_lib.sh):
#   scripts/build_variant.sh NAME "-DFOO=1 ..." [SRC_DIR]
# SRC_DIR defaults to paper_2009_14514_b200/csrc; objects under build/variants/NAME/.
cd "$(dirname $0)/.."
NAME=$1; EXTRA=$2; SRC=${3:-paper_2009_14514_b200/csrc}
OUT=build/variants/$NAME; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in grid levels wcsph pcisph halo; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 $ARCH -lineinfo --fmad=false -Xcompiler -fPIC,-O3 \
    -Xptxas -v $EXTRA -I include -I paper_2009_14514_b200/csrc -c $SRC/$f.cu -o $OUT/$f.o \
    2> $OUT/$f.ptxas.txt || { cat $OUT/$f.ptxas.txt; exit 1; } &
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -o build/variants/$NAME.so $OUT/*.o -cudart static
grep -A3 "k_refresh" $OUT/pcisph.ptxas.txt | grep -E "spill|Used" | head -4
