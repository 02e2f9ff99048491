#!/bin/bash
# Build libgfb.so variants that differ only in the star-pair TMA tile
# (experiments; the production build is csrc/Makefile). Output:
# build/variants/libgfb_<name>.so
set -e
cd "$(dirname "$0")/../paper_2509_02197_b200/csrc"
make -s
mkdir -p ../../build/variants
OBJS=$(ls ../../build/obj/*.o | grep -v star_tma.o)
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
    -c star_tma.cu -o ../../build/variants/star_tma_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/libgfb_$name.so $OBJS \
    ../../build/variants/star_tma_$name.o -lcudart
}
build t32r4u1 -DGFB_STAR_TPY=32 -DGFB_STAR_KR=4 -DGFB_STAR_UNROLL=1 &
build t32r4u0 -DGFB_STAR_TPY=32 -DGFB_STAR_KR=4 -DGFB_STAR_UNROLL=0 &
build t16r2u1 -DGFB_STAR_TPY=16 -DGFB_STAR_KR=2 -DGFB_STAR_UNROLL=1 &
build t32r2u1 -DGFB_STAR_TPY=32 -DGFB_STAR_KR=2 -DGFB_STAR_UNROLL=1 &
build t16r4u1 -DGFB_STAR_TPY=16 -DGFB_STAR_KR=4 -DGFB_STAR_UNROLL=1 &
build t32r4u1m32 -DGFB_STAR_TPY=32 -DGFB_STAR_KR=4 -DGFB_STAR_UNROLL=1 -DGFB_STAR_TPM=32 &
wait
ls ../../build/variants/*.so
