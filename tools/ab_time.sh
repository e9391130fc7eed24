#!/bin/bash
# A/B timing of dev builds (tools/dev/<name>/libctfiss.so; "main" = the
# regular paper_2510_02382_b200/libctfiss.so) on one config:
#   tools/ab_time.sh "<prof_cfg args>" name1 name2 ...   (two alternating rounds)
ARGS=$1; shift
for round in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then LIBV=; else LIBV=tools/dev/$n/libctfiss.so; fi
    echo -n "$n: "; CTF_DEV_LIB=$LIBV timeout 300 python tools/prof_cfg.py $ARGS 2>&1 | tail -1
  done
done
