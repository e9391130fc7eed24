for c in 2; do timeout 300 python tools/prof_cfg.py --cfg $c --prec f32 --iters 6 2>&1 | tail -1; done
