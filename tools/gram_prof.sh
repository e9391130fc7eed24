timeout 600 python tools/prof_cfg.py --cfg 3 --prec f32 --iters 3 --mixtures 16 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "trajectory" 2>&1 | tail -2
