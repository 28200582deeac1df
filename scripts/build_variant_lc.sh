#!/bin/bash
# Like build_variant.sh, for lora_compose.cu: scripts/build_variant_compose.sh NAME "FLAGS"
set -e
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=$2
C=paper_2603_22276_b200/csrc
make -s -C $C
mkdir -p variants/obj_$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -Iinclude -I$C/kernels $FLAGS -c $C/kernels/lora_compose.cu -o variants/obj_$NAME/lora_compose.o
OBJS=$(ls $C/obj/*.o $C/obj/kernels/*.o | grep -v "/lora_compose.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libdfx_$NAME.so $OBJS variants/obj_$NAME/lora_compose.o -lcudart
echo built variants/libdfx_$NAME.so
