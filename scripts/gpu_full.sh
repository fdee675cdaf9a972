nproc
timeout -s KILL 1200 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=5 2>&1 | tail -12
