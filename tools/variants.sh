#!/bin/bash
# time every compiled variant for one config: tools/variants.sh <cfg> <prec> <rmax> "v1 v2 ..."
cfg=$1; prec=$2; shift 2
for v in "$@"; do CTF_SWEEP_VARIANT=$v python tools/prof_cfg.py --cfg $cfg --prec $prec --iters 5 2>&1 | tail -2; done
