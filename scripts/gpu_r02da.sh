# round 2: one host pool per compress part (two half-size pools)
export CUDA_MODULE_LOADING=EAGER
for rep in 1 2 3; do timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 1,3p; done
timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | sed -n 2,3p
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02da_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02da_tests.log
