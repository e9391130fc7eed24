CTF_GRAM_LEAN=1 timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 10 2>&1 | tail -2
CTF_GRAM_LEAN=0 timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 10 2>&1 | tail -1
