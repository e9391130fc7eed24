#!/bin/bash
for p in f32 f64; do timeout 300 python tools/prof_cfg.py --cfg 0 --prec $p --iters 50 2>&1 | tail -1; done
timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 5 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
