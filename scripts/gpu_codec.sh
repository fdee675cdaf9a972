timeout -s KILL 600 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -5
FC_TRACE=0 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | tail -6
FC_COMPRESS_SPLIT=0 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep "^compress" | tail -1
