# round 2: compress = whole-batch Gram/select + staged assembly parts (turn order A then B) on child streams; sweep, codec tests
export CUDA_MODULE_LOADING=EAGER
for S in 1 2 3 4 6 8; do echo "split $S"; FC_COMPRESS_SPLIT=$S timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 3p; done
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_capi.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02az_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02az_tests.log
