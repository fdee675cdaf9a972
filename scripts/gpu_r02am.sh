# round 2: stream-ordered decompress APIs (one H2D, no host sync), codec tests + codec bench
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_capi.py tests/test_cli.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02am_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02am_tests.log
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-scoring --no-engine --no-cpu > gpurun_out/r02am_bench.json 2> gpurun_out/r02am_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02am_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02am_bench.json')); print(d['value']); print('codec', {k: d['codec'][k] for k in ('compress_GBps','compress_frac_hbm','decompress_GBps_e2e','decompress_frac_hbm_e2e')}, d['codec']['roofline']); print('large', {k: d['codec_large'][k] for k in ('compress_frac_hbm','decompress_frac_hbm_e2e')})"
