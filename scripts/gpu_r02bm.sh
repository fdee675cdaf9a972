# round 2: parallel snapshot load (framing pass, CRC + import per record on child streams, in-order apply); store/snapshot tests; config[4] checkpoint numbers
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_snapshot.py tests/test_gpu_store.py tests/test_cli.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02bm_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02bm_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-scoring --no-engine --no-cpu > gpurun_out/r02bm_bench.json 2> gpurun_out/r02bm_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02bm_bench.json')); print(d['codec_large']['checkpoint'])"
