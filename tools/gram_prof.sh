CTF_SWEEP_VARIANT=32,2,4,512 timeout 600 python tools/prof_cfg.py --cfg 3 --prec f32 --iters 3 --mixtures 16 2>&1 | tail -2
