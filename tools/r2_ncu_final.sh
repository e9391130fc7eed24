#!/bin/bash
# End-of-round ncu --set full captures (one kernel each, after the plain runs exited 0), summarised
# on the box: the fp64 cfg1 covariance kernel, lambda_kernel and the MU-V partial kernel on cfg1 fp64,
# mub_kernel and the frame-split kernel on 16 cfg3 mixtures.
O=gpurun_out/ncu_final; mkdir -p $O
cap() {  # name regex tfbins prof_cfg-args...
  local name=$1 rx=$2 n=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s 2 -c 1 -o $O/$name -f python tools/prof_cfg.py "$@" > $O/$name.log 2>&1
  echo "$name rc=$?"
  [ -f $O/$name.ncu-rep ] || return
  python tools/ncu_lines.py $O/$name.ncu-rep 40 > $O/$name.lines.txt 2>&1
  python tools/ncu_summary.py $O/$name.ncu-rep "$name" "ncu --set full --import-source on --clock-control none -k regex:$rx -s 2 -c 1 python tools/prof_cfg.py $*" "$name" $n > $O/$name.summary.json 2>&1
  rm -f $O/$name.ncu-rep
}
cap gram_kernel_f64 gram_kernel 32832000 --cfg 1 --prec f64 --iters 3
cap lambda_kernel_f64 lambda_kernel 32832000 --cfg 1 --prec f64 --iters 3
cap muv_partial_kernel_f64 muv_partial 32832000 --cfg 1 --prec f64 --iters 3
cap mub_kernel_c3 mub_kernel 32784000 --cfg 3 --mixtures 16 --iters 3
cap fsplit_kernel_c3 fsplit_kernel 32784000 --cfg 3 --mixtures 16 --iters 3
ls -la $O
