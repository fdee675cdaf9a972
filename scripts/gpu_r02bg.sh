# round 2: parallel pwrite snapshot save + sized read on load; snapshot/codec/engine tests; config[4] bench section
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_snapshot.py tests/test_gpu_codec.py tests/test_engine.py tests/test_cli.py tests/test_gpu_store.py -q -x -m gpu > gpurun_out/r02bg_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02bg_tests.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-codec --no-scoring --no-engine --no-cpu > gpurun_out/r02bg_bench.json 2> gpurun_out/r02bg_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02bg_bench.json')); print(d['codec_large'])"
