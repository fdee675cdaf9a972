export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=2 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep -E "^\[compress\]|^compress" | tail -30
