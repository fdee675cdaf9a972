# round 2: engine speculation, snapshot CRC, fused scoring (warp-aggregated histogram) — tests + timings
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1200 python -m pytest tests/test_engine.py tests/test_gpu_snapshot.py tests/test_gpu_store.py tests/test_cli.py -q -x > gpurun_out/r02z_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02z_tests.log
timeout -s KILL 300 python scripts/time_store.py 100000 gets > gpurun_out/r02z_store_time.log 2>&1; cat gpurun_out/r02z_store_time.log
FC_ENGINE_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-scoring --mixed-requests 16384 > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02z_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02z_bench.json')); print('large', d.get('codec_large')); print('engine', d['engine'])"
