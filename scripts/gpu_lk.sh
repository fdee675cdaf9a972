export CUDA_MODULE_LOADING=EAGER
for r in 32 64; do echo "refresh $r"; FC_SHORTLIST_REFRESH=$r FC_SHORTLIST_DEBUG=16 timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -2; done
