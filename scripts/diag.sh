for r in 100000 300000; do for k in 32 64; do timeout -s KILL 100 python scripts/dbg2.py $r $k 4096 || echo "$r $k fail"; done; done
timeout -s KILL 100 python scripts/dbg2.py 1000000 32 1024 || echo "1M 32 1024 fail"
timeout -s KILL 100 python scripts/dbg2.py 1000000 32 4096 || echo "1M 32 4096 fail"
