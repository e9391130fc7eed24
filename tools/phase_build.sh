#!/bin/bash
# Instrumented build for tools/phase_timing.py: ctf_sweep_gram.cu with
# -DCTF_PHASE_TIMING linked with the regular objects into tools/phase/libctfiss.so
set -e
cd "$(dirname "$0")/../paper_2510_02382_b200/csrc"
make -s
mkdir -p ../../tools/phase
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DCTF_PHASE_TIMING -c ctf_sweep_gram.cu -o ../../tools/phase/ctf_sweep_gram_phase.o
OBJS=$(ls build/*.o | grep -v ctf_sweep_gram.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/phase/libctfiss.so $OBJS \
  ../../tools/phase/ctf_sweep_gram_phase.o -cudart=static -ldl -lpthread
