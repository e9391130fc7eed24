#!/bin/bash
# one ncu --set full capture of the default frame-split kernel on cfg4 (1 mixture)
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fs_c4.log 2>&1 && tail -1 gpurun_out/fs_c4.log && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fsplit_kernel -s 2 -c 1 -o gpurun_out/fsplit_c4_cs8 -f python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fsplit_ncu.log 2>&1; tail -2 gpurun_out/fsplit_ncu.log
