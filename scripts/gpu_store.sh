timeout -s KILL 300 python scripts/time_store.py 100000 2>&1 | tail -8
