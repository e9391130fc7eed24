timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for c in 0 1; do for pr in f32 f64; do timeout 300 python tools/prof_cfg.py --cfg $c --prec $pr --iters 5 --rule ip 2>&1 | tail -1; done; done
