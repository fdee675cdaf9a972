timeout -s KILL 900 python -m pytest tests/test_engine.py -q -x 2>&1 | tail -3
FC_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-codec --no-scoring > gpurun_out/bench_eng.json 2>gpurun_out/bench_eng.err; echo rc=$?; grep "\[engine\]" gpurun_out/bench_eng.err | tail -3; python -c "import json; print(json.load(open('gpurun_out/bench_eng.json'))['engine'])"
