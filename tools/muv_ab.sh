#!/bin/bash
# A/B of MU-V partial kernel variants (tools/dev_build_tu.sh NAME ctf_capi -D...):
#   tools/muv_ab.sh name1 name2 ...   ("main" = the regular library), cfg1 in both precisions,
#   two alternating rounds; the "mu" figure is MU-V + reduce/apply per iteration
for round in 1 2; do
  for prec in f64 f32; do
    for n in "$@"; do
      if [ "$n" = main ]; then LIBV=; else LIBV=tools/dev/$n/libctfiss.so; fi
      echo -n "$n: "; CTF_DEV_LIB=$LIBV timeout 300 python tools/prof_cfg.py --cfg 1 --prec $prec --iters 10 2>&1 | tail -1
    done
  done
done
