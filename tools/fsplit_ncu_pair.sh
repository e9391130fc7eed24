#!/bin/bash
# ncu --set full (source lines) of the cfg4 frame-split kernel, one step per
# exchange (pair=0) and step pairs (pair=1), 1 mixture
mkdir -p gpurun_out
for pair in 0 1; do
  CTF_FSPLIT_PAIR=$pair timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fs_c4_p$pair.log 2>&1 && tail -1 gpurun_out/fs_c4_p$pair.log && \
  CTF_FSPLIT_PAIR=$pair timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fsplit_kernel -s 2 -c 1 -o gpurun_out/fsplit_c4_p$pair -f python tools/prof_cfg.py --cfg 4 --mixtures 1 --iters 1 > gpurun_out/fsplit_ncu_p$pair.log 2>&1; tail -2 gpurun_out/fsplit_ncu_p$pair.log
done
