timeout -s KILL 900 python -m pytest tests/test_cli.py tests/test_engine.py -q -x 2>&1 | tail -15
