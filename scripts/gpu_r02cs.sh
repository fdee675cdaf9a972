export CUDA_MODULE_LOADING=EAGER
FC_TRACE=1 timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep "\[gap\]" | tail -12
