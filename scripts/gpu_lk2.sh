timeout -s KILL 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py tests/test_engine.py -q -x -m gpu 2>&1 | tail -2
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-codec --no-scoring --no-engine > gpurun_out/bench_lk.json 2>gpurun_out/bench_lk.err
python -c "import json; d=json.load(open('gpurun_out/bench_lk.json')); print(d['value'], d['ms_per_step_all'][:8], d['kernel_ms'], d['clocks'])"
