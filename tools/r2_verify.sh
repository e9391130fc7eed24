#!/bin/bash
# Round-2 measurement pass on one B200: GPU test suite, smoke, the default
# bench line (cfg1 f64 + the f32 line), the reference arm, the launch list of
# the default bench and one ncu --set full capture of the cfg1 f64 kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
[ "$SKIP_NCU" = 1 ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-frontend --no-f32 > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gram_kernel -s 2 -c 1 -o gpurun_out/gram_c1_f64_full -f \
  python tools/prof_cfg.py --cfg 1 --prec f64 --iters 2 > gpurun_out/gram_f64_full.log 2>&1; echo "ncu gram f64 rc=$?"
ls -la gpurun_out
