python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; tail -2 gpurun_out/bench_f32.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_bench_f32.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-frontend > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
