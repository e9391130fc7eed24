#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fsplit.py -x -q 2>&1 | tail -2
for ag in 0 1; do
  CTF_FSPLIT_AG=$ag CTF_SWEEP_VARIANT=60,2,32,256 timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -1
  for v in 32,4,16,128 32,2,16,128; do
    CTF_FSPLIT_AG=$ag CTF_SWEEP_VARIANT=$v timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 2 2>&1 | tail -1
  done
done
