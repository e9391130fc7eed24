#!/bin/bash
# Timing of the lambda-ahead path (lambda_kernel + 16-byte copies of 1/lambda in
# the covariance-domain kernel's prologue; per variant by gram_lpre()): the
# regular build, and the iteration kernel alone (CTF_DEV_SKIP_LAMBDA=1: stale
# 1/lambda after two iterations, timing only), two rounds per config.
# Builds with -DCTF_GRAM_LPRE=0 / 1 (tools/dev_build.sh) give the other arm.
run() { echo -n "$1 [$2]: "; env $1 timeout 300 python tools/prof_cfg.py $2 2>&1 | tail -1; }
for round in 1 2; do
  for a in "--cfg 1 --prec f64 --iters 10" "--cfg 1 --prec f32 --iters 10" "--cfg 2 --prec f32 --mixtures 32 --iters 5"; do
    run X=1 "$a"; run CTF_DEV_SKIP_LAMBDA=1 "$a"
  done
done
