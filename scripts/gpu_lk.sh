export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup.py -q -x -m gpu 2>&1 | tail -2
timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1
FC_SHORTLIST_DEBUG=16 timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -2
