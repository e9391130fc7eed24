timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python bench.py --cfg 3 --no-frontend > gpurun_out/b_c3_f32.json 2>gpurun_out/b_c3.err; tail -1 gpurun_out/b_c3.err
