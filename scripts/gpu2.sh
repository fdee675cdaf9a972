timeout -s KILL 400 python -m pytest tests/test_gpu_codec.py tests/test_gpu_store.py -q -m gpu 2>&1 | tail -40
timeout -s KILL 300 python -m pytest tests/test_gpu_lookup.py -q -m gpu 2>&1 | tail -30
