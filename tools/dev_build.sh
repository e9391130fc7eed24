#!/bin/bash
# Dev build for A/B timing of one gram_kernel variant: ctf_sweep_gram.cu with
# only that variant (CTF_GRAM_DEV="M L NT FT", default "2 5 256 4"; fp64/IP lists empty), linked
# with the regular objects into tools/dev/<name>/libctfiss.so (-DCTF_DEV_F64: the
# fp64 variant of that shape instead). Use it with
#   CTF_DEV_LIB=tools/dev/<name>/libctfiss.so python tools/prof_cfg.py ...
# Extra nvcc flags (e.g. -DCTF_PHASE_TIMING) after the name.
set -e
NAME=${1:-dev}; shift || true
read DM DL DNT DFT <<< "${CTF_GRAM_DEV:-2 5 256 4}"
cd "$(dirname "$0")/../paper_2510_02382_b200/csrc"
# (expects the regular objects in build/: run make first)
D=../../tools/dev/$NAME
mkdir -p $D
SRC=${DEV_FILE:-ctf_sweep_gram}  # DEV_FILE=ctf_sweep_fsplit: the frame-split variants instead
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -v -DCTF_GRAM_DEV -DCTF_DEV_M=$DM -DCTF_DEV_L=$DL -DCTF_DEV_NT=$DNT -DCTF_DEV_FT=$DFT "$@" -c $SRC.cu -o $D/gram.o 2> $D/ptxas.log
grep -A2 "_kernel" $D/ptxas.log | grep -E "spill|Used" | head -4
OBJS=$(ls build/*.o | grep -v $SRC.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libctfiss.so $OBJS $D/gram.o -cudart=static -ldl -lpthread
