export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep "exact-difference" | tail -2
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | grep "exact-difference" | tail -1
