python bench.py > gpurun_out/bench_f32.json 2>/dev/null
python bench.py --cfg 0 --dtype f64 --no-frontend > gpurun_out/b_c0_f64.json 2>/dev/null
python bench.py --cfg 0 --dtype f32 --no-frontend > gpurun_out/b_c0_f32.json 2>/dev/null
python bench.py --cfg 1 --dtype f64 --no-frontend > gpurun_out/b_c1_f64.json 2>/dev/null
python bench.py --cfg 2 --dtype f32 --no-frontend > gpurun_out/b_c2_f32.json 2>/dev/null
python bench.py --cfg 4 --dtype f32 --no-frontend --no-e2e --steps 3 > gpurun_out/b_c4_f32.json 2>/dev/null
python bench.py --impl reference > gpurun_out/bench_reference.json 2>/dev/null
ls -la gpurun_out/*.json
