# round 2: K7 split + L2 bulk prefetch of each block frame ranges
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | head -3
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_capi.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02be_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02be_tests.log
