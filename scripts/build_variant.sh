#!/bin/bash
# Builds an experiment variant of libdfx.so with extra nvcc flags for norm_tc.cu only:
#   scripts/build_variant.sh NAME "-DDFX_KO_MMA ..."   ->  variants/libdfx_NAME.so
# (knock-out / tuning experiments; run with DFX_LIB=variants/libdfx_NAME.so)
set -e
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=$2
C=paper_2603_22276_b200/csrc
make -s -C $C
mkdir -p variants/obj_$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -Iinclude -I$C/kernels $FLAGS -c $C/kernels/norm_tc.cu -o variants/obj_$NAME/norm_tc.o
OBJS=$(ls $C/obj/*.o $C/obj/kernels/*.o | grep -v norm_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libdfx_$NAME.so $OBJS variants/obj_$NAME/norm_tc.o -lcudart
echo built variants/libdfx_$NAME.so
