#!/bin/bash
# Build an experimental variant of libsymdist_b200.so with extra nvcc defines.
# Usage: tools/build_variant.sh <name> "-DSDB_TILE_BLOCKS=2 ..."
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
OUT=paper_2408_10743_b200/_variants/$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in kernels prep; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 $ARCH -lineinfo $DEFS -Xcompiler -fPIC -c paper_2408_10743_b200/csrc/$f.cu -o $OUT/$f.o
done
for f in gf2 packages comm tcenc engine capi; do
  g++ -O3 -std=c++17 -fPIC $DEFS -I/usr/local/cuda/include -c paper_2408_10743_b200/csrc/$f.cpp -o $OUT/$f.o
done
/usr/local/cuda/bin/nvcc $ARCH -shared -o $OUT/libsymdist_b200.so $OUT/kernels.o $OUT/prep.o $OUT/gf2.o $OUT/packages.o $OUT/comm.o $OUT/tcenc.o $OUT/engine.o $OUT/capi.o -lpthread -ldl
echo $OUT/libsymdist_b200.so
