#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fsplit.py -x -q 2>&1 | tail -3
timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -1
CTF_SWEEP_VARIANT=60,2,32,256 CTF_SWEEP_KIND=5 timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 4 --iters 2 2>&1 | tail -1
CTF_SWEEP_KIND=5 CTF_SWEEP_VARIANT=32,2,16,256 timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 2 2>&1 | tail -1
CTF_SWEEP_KIND=5 CTF_SWEEP_VARIANT=32,2,16,128 timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 2 2>&1 | tail -1
timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fs_c4.log 2>&1 && tail -1 gpurun_out/fs_c4.log && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fsplit_kernel -s 2 -c 1 -o gpurun_out/fsplit_c4_sweep -f python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fsplit_ncu.log 2>&1; tail -2 gpurun_out/fsplit_ncu.log
