#!/bin/bash
timeout 300 python tools/prof_cfg.py --cfg 0 --prec f32 --iters 3 2>&1 | tail -1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:reduce_apply -s 3 -c 1 -o gpurun_out/apply_c0 -f python tools/prof_cfg.py --cfg 0 --prec f32 --iters 3 > gpurun_out/apply_ncu.log 2>&1; tail -1 gpurun_out/apply_ncu.log
