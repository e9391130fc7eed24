#!/bin/bash
# Round-1 final measurement: every BASELINE config's bench line, the reference
# arm, the cfg1 launch list and one ncu --set full capture of the cfg1 kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; echo "cfg1 f32 rc=$?"
python bench.py --cfg 1 --dtype f64 --no-frontend > gpurun_out/b_c1_f64.json 2>/dev/null; echo "cfg1 f64 rc=$?"
python bench.py --cfg 0 --dtype f64 --no-frontend > gpurun_out/b_c0_f64.json 2>/dev/null; echo "cfg0 f64 rc=$?"
python bench.py --cfg 0 --dtype f32 --no-frontend > gpurun_out/b_c0_f32.json 2>/dev/null; echo "cfg0 f32 rc=$?"
python bench.py --cfg 2 --dtype f32 --no-frontend > gpurun_out/b_c2_f32.json 2>/dev/null; echo "cfg2 rc=$?"
timeout 900 python bench.py --cfg 3 --dtype f32 --no-frontend --steps 5 > gpurun_out/b_c3_f32.json 2>/dev/null; echo "cfg3 rc=$?"
timeout 900 python bench.py --cfg 4 --dtype f32 --no-frontend --steps 3 > gpurun_out/b_c4_f32.json 2>/dev/null; echo "cfg4 rc=$?"
python bench.py --impl reference > gpurun_out/bench_reference.json 2>/dev/null; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_bench_f32.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-frontend > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gram_kernel -s 2 -c 1 -o gpurun_out/gram_c1_full -f \
  python tools/prof_cfg.py --cfg 1 --prec f32 --iters 2 > gpurun_out/gram_full.log 2>&1; echo "ncu gram rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fsplit_kernel -s 2 -c 1 -o gpurun_out/fsplit_c3_full -f \
  python tools/prof_cfg.py --cfg 3 --mixtures 8 --iters 2 > gpurun_out/fsplit_full.log 2>&1; echo "ncu fsplit rc=$?"
ls -la gpurun_out
