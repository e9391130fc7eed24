#!/bin/bash
timeout 300 python tools/prof_cfg.py --cfg 0 --prec f32 --iters 3 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_cfg.py --cfg 0 --prec f32 --iters 3 > gpurun_out/c0_launches.csv 2>&1; grep -E "kernel" gpurun_out/c0_launches.csv | awk -F'","' '{print $5, $(NF)}' | tail -12
