#!/bin/bash
for i in 1 2; do timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 10 2>&1 | tail -1; done
timeout 300 python tools/prof_cfg.py --cfg 1 --prec f64 --iters 5 2>&1 | tail -1
timeout 300 python tools/prof_cfg.py --cfg 2 --mixtures 32 --iters 3 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
