#!/bin/bash
# A/B over the three covariance-kernel configs: tools/ab3.sh name1 name2 ...
# ("main" = the regular library, others tools/dev/<name>/libctfiss.so), two alternating rounds
for round in 1 2; do
  for a in "--cfg 1 --prec f64 --iters 10" "--cfg 1 --prec f32 --iters 10" "--cfg 2 --prec f32 --mixtures 32 --iters 5"; do
    for n in "$@"; do
      if [ "$n" = main ]; then LIBV=; else LIBV=tools/dev/$n/libctfiss.so; fi
      echo -n "$n: "; CTF_DEV_LIB=$LIBV timeout 300 python tools/prof_cfg.py $a 2>&1 | tail -1
    done
  done
done
