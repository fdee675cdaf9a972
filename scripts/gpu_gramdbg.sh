for m in 0 3; do echo "dbg $m"; FC_COMPRESS_SPLIT=1 FC_GRAM_DBG=$m timeout -s KILL 120 python scripts/time_codec.py 256 2>&1 | grep -o "'gram': [0-9.]*" | tail -1; done
timeout -s KILL 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -2
