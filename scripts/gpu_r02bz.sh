# round 2: Gram work-item split for few tiles (config[4], engine flushes); timing + codec/engine tests
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | head -3
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_engine.py tests/test_capi.py -q -x -m gpu > gpurun_out/r02bz_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02bz_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-scoring --no-cpu --mixed-requests 4096 > /tmp/b.json 2> /tmp/b.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('/tmp/b.json')); print('large', {k: d['codec_large'][k] for k in ('compress_frac_hbm','compress_s')}, 'engine', d['engine']['requests_per_s'], d['engine']['mixed']['requests_per_s'])"
