timeout 900 python -m pytest tests/test_gpu_stft.py -q -x 2>&1 | tail -2
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fe.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/fe.json')); f=d['frontend']; print(f['stft'], f['istft'], f['round_trip_max_rel_err'])"
