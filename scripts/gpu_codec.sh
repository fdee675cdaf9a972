timeout -s KILL 600 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -2
for k in 1 2 3 4; do echo "split $k"; FC_COMPRESS_SPLIT=$k timeout -s KILL 100 python scripts/time_codec.py 256 2>&1 | grep "^compress" | tail -2; done
