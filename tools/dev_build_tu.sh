#!/bin/bash
# Dev build of one translation unit with extra flags for A/B timing:
#   tools/dev_build_tu.sh NAME TU [nvcc flags...]   (TU without .cu, e.g. ctf_capi)
# links it with the regular objects into tools/dev/NAME/libctfiss.so; use with
#   CTF_DEV_LIB=tools/dev/NAME/libctfiss.so python tools/prof_cfg.py ...
set -e
NAME=$1; TU=$2; shift 2
cd "$(dirname "$0")/../paper_2510_02382_b200/csrc"
D=../../tools/dev/$NAME
mkdir -p $D
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -v "$@" -c $TU.cu -o $D/$TU.o 2> $D/ptxas.log
OBJS=$(ls build/*.o | grep -v /$TU.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libctfiss.so $OBJS $D/$TU.o -cudart=static -ldl -lpthread
