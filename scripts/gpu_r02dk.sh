# round 2: pinned staging of the lookup APIs' host outputs — lookup/decide/engine tests + bench (e2e)
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_lookup_i8.py tests/test_engine.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02dk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02dk_tests.log
timeout -s KILL 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02dk_bench.json 2> gpurun_out/r02dk_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r02dk_bench.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
