#!/bin/bash
# cfg2 geometry: frame-split cluster variants vs the covariance kernel
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg.py --cfg 2 --mixtures 16 --iters 2 2>&1 | tail -1
for v in 12,4,6,256 12,2,12,256 12,4,12,128; do
  CTF_SWEEP_KIND=5 CTF_SWEEP_VARIANT=$v timeout 300 python tools/prof_cfg.py --cfg 2 --mixtures 16 --iters 2 2>&1 | tail -2
done
