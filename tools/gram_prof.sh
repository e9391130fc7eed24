for c in 0 1 2; do timeout 300 python tools/prof_cfg.py --cfg $c --prec f32 --iters 10 2>&1 | tail -1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or trajectory or odd or covariance" 2>&1 | tail -2
