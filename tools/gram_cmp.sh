# dev: gram_kernel vs frame-domain sweep (CTF_SWEEP_KIND=0) timing, then fp32 parity tests
for c in 0 1 2; do
  timeout 300 python tools/prof_cfg.py --cfg $c --prec f32 --iters 10 2>&1 | tail -2
  CTF_SWEEP_KIND=0 timeout 300 python tools/prof_cfg.py --cfg $c --prec f32 --iters 10 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f32 or fp32 or cfg1 or cfg2 or sharded or odd or batch or determin" 2>&1 | tail -15
