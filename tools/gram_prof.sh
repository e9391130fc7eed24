CTF_SWEEP_KIND=0 timeout 300 python tools/prof_cfg.py --cfg 0 --prec f64 --iters 10 2>&1 | tail -1
timeout 300 python tools/prof_cfg.py --cfg 0 --prec f64 --iters 10 2>&1 | tail -1
CTF_SWEEP_KIND=0 timeout 300 python tools/prof_cfg.py --cfg 0 --prec f32 --iters 10 2>&1 | tail -1
timeout 300 python tools/prof_cfg.py --cfg 0 --prec f32 --iters 10 2>&1 | tail -1
