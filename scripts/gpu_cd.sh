export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_store.py tests/test_gpu_lookup.py -q -x -m gpu 2>&1 | tail -3
FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 2>&1 | tail -14
