FC_TRACE=1 timeout -s KILL 300 python scripts/time_store.py 100000 gets 2>&1 | tail -5
timeout -s KILL 600 python -m pytest tests/test_gpu_store.py -q -x 2>&1 | tail -3
