#!/bin/bash
# full GPU suite, then the cfg3 / cfg4 bench lines on the frame-split kernel
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --cfg 3 --dtype f32 --no-frontend --steps 5 > gpurun_out/b_c3_f32.json 2>gpurun_out/b_c3.err; tail -c 600 gpurun_out/b_c3_f32.json
timeout 900 python bench.py --cfg 4 --dtype f32 --no-frontend --steps 3 > gpurun_out/b_c4_f32.json 2>gpurun_out/b_c4.err; tail -c 600 gpurun_out/b_c4_f32.json
