for k in 2 3 4 6; do for st in 0 1; do echo "split $k stagger $st"; FC_COMPRESS_STAGGER=$st FC_COMPRESS_SPLIT=$k timeout -s KILL 100 python scripts/time_codec.py 256 2>&1 | grep "^compress" | tail -2; done; done
timeout -s KILL 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -2
