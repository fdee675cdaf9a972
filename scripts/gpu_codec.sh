for k in 1 2 3 4 8; do echo "split $k"; FC_COMPRESS_SPLIT=$k timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep "^compress" | tail -2; done
