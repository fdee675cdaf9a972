timeout -s KILL 600 python -m pytest tests/test_gpu_snapshot.py -q -x 2>&1 | tail -25
