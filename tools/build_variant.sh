#!/bin/bash
# build_variant.sh <csrc_dir> <out.so> : build the library from an alternative
# source tree (A/B experiments; load with SA_LIB_PATH=<out.so>)
set -e
SRC=$1; OUT=$2; OBJ=$(mktemp -d)
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC"
for f in sa_abi sa_d1 sa_d2 sa_d3 sa_scan sa_meshgen sa_host; do nvcc $FL -c -o $OBJ/$f.o $SRC/$f.cu & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJ/*.o
rm -rf $OBJ
