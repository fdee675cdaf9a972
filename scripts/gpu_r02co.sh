# round 2: grouped decompress split over frame slices when jobs are few (config[4]); codec tests
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | tail -2
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | tail -2
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02co_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02co_tests.log
