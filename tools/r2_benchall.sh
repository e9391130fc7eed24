#!/bin/bash
# Round-2 measurement pass on one B200: every BASELINE config's bench line,
# the reference arm, the default bench's launch list and ncu --set full
# captures of the dominant kernels (each only after its plain run exited 0).
mkdir -p gpurun_out/r2
O=gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err; echo "cfg1 (f64 + f32) rc=$?"
timeout 600 python bench.py --cfg 0 --dtype f64 --no-frontend > $O/b_c0_f64.json 2>/dev/null; echo "cfg0 f64 rc=$?"
timeout 600 python bench.py --cfg 0 --dtype f32 --no-frontend > $O/b_c0_f32.json 2>/dev/null; echo "cfg0 f32 rc=$?"
timeout 900 python bench.py --cfg 2 --no-frontend > $O/b_c2_f32.json 2>/dev/null; echo "cfg2 rc=$?"
timeout 900 python bench.py --cfg 3 --no-frontend --steps 5 > $O/b_c3_f32.json 2>/dev/null; echo "cfg3 rc=$?"
timeout 900 python bench.py --cfg 4 --no-frontend --steps 3 > $O/b_c4_f32.json 2>/dev/null; echo "cfg4 rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2>/dev/null; echo "ref rc=$?"
[ "$SKIP_NCU" = 1 ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_c1_f64.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-frontend --no-f32 > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gram_kernel -s 2 -c 1 -o $O/gram_c1_f64 -f \
  python tools/prof_cfg.py --cfg 1 --prec f64 --iters 2 > $O/gram_c1_f64.log 2>&1; echo "ncu gram f64 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gram_kernel -s 2 -c 1 -o $O/gram_c2_f32 -f \
  python tools/prof_cfg.py --cfg 2 --mixtures 32 --iters 2 > $O/gram_c2_f32.log 2>&1; echo "ncu gram cfg2 rc=$?"
# reports are summarised on the box (gpurun_out is copied back only below 64 MiB)
for r in gram_c1_f64 gram_c2_f32; do
  [ -f $O/$r.ncu-rep ] || continue
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  python tools/ncu_lines.py $O/$r.ncu-rep 60 > $O/$r.lines.txt 2>&1
  n=32832000; [ $r = gram_c2_f32 ] && n=65600000
  python tools/ncu_summary.py $O/$r.ncu-rep "$r" "ncu --set full -k regex:gram_kernel -s 2 -c 1 (tools/r2_benchall.sh)" "$r" $n > $O/$r.summary.json 2>&1
  rm -f $O/$r.ncu-rep
done
ls -la $O
