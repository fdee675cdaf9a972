timeout -s KILL 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_store.py -q -x 2>&1 | tail -2
for g in 0 1; do echo "groups $g"; FC_DEC_GROUPS=$g timeout -s KILL 100 python scripts/time_codec.py 256 2>&1 | grep "^decompress"; done
