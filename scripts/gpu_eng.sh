timeout -s KILL 900 python -m pytest tests/test_engine.py tests/test_gpu_lookup.py -q -x 2>&1 | tail -2
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-cpu --no-codec --no-scoring > gpurun_out/bench_eng.json 2>gpurun_out/bench_eng.err
python -c "import json; d=json.load(open('gpurun_out/bench_eng.json')); e=d['engine']; print(e['requests_per_s'], e['index_stats'], e['mixed']['requests_per_s'])"
