#!/bin/bash
# Builds libdfx.so with norm_tc.cu replaced by another source (A/B of kernel versions):
#   scripts/build_variant_src.sh NAME path/to/norm_tc.cu ["-DFLAGS"]  ->  variants/libdfx_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; FLAGS=$3
C=paper_2603_22276_b200/csrc
make -s -C $C
mkdir -p variants/obj_$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -Iinclude -I$C/kernels $FLAGS -c $SRC -o variants/obj_$NAME/norm_tc.o
OBJS=$(ls $C/obj/*.o $C/obj/kernels/*.o | grep -v norm_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libdfx_$NAME.so $OBJS variants/obj_$NAME/norm_tc.o -lcudart
echo built variants/libdfx_$NAME.so
