#!/bin/bash
# A/B of the frame-split step schedules (one ISS step per exchange vs step
# pairs) on cfg3 / cfg4, alternating runs on one box.
mkdir -p gpurun_out
for rep in 1 2; do
  for pair in 0 1; do
    CTF_FSPLIT_PAIR=$pair timeout 300 python tools/prof_cfg.py --cfg 4 --mixtures 8 --iters 3 2>&1 | tail -1 | sed "s/^/pair=$pair /"
    CTF_FSPLIT_PAIR=$pair timeout 300 python tools/prof_cfg.py --cfg 3 --mixtures 16 --iters 3 2>&1 | tail -1 | sed "s/^/pair=$pair /"
  done
done
