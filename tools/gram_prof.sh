for c in 1 2; do timeout 300 python tools/prof_cfg.py --cfg $c --prec f32 --iters 6 2>&1 | tail -1; done
timeout 300 python tools/prof_cfg.py --cfg 1 --prec f64 --iters 4 2>&1 | tail -1
