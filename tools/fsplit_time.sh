#!/bin/bash
mkdir -p gpurun_out
for v in 60,2,32,256 60,4,20,128; do
  CTF_SWEEP_KIND=5 CTF_FSPLIT_AG=0 CTF_SWEEP_VARIANT=$v timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -2
done
