#!/bin/bash
# frame-split cluster kernel: parity, then cfg3/cfg4 timing against the alternatives
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fsplit.py -x -q 2>&1 | tail -25 > gpurun_out/fsplit_tests.log
cat gpurun_out/fsplit_tests.log
for v in "" ; do :; done
timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -2
CTF_SWEEP_VARIANT=60,2,32,256 CTF_SWEEP_KIND=5 timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -2
CTF_SWEEP_KIND=2 timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -1
timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 2 2>&1 | tail -1
for v in 32,2,16,128 32,2,16,256 32,1,16,128; do
  CTF_SWEEP_KIND=5 CTF_SWEEP_VARIANT=$v timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 2 2>&1 | tail -2
done
