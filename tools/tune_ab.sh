#!/bin/bash
# A/B of Gram task layouts (CTF_GRAM_TUNE) on cfg1 fp32
for round in 1 2; do
  echo -n "default: "; timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 10 2>&1 | tail -1
  for f in "$@"; do
    echo -n "$f: "; CTF_GRAM_TUNE="$(cat $f)" timeout 300 python tools/prof_cfg.py --cfg 1 --prec f32 --iters 10 2>&1 | tail -1
  done
done
