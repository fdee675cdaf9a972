for m in 0 1 2 3; do echo "dbg $m"; FC_GRAM_DBG=$m timeout -s KILL 120 python scripts/time_codec.py 256 2>&1 | grep -o "'gram': [0-9.]*" | tail -1; done
