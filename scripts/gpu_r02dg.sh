# round 2: compress host timeline (FC_TRACE) + kernel breakdown, config[2] batch
export CUDA_MODULE_LOADING=EAGER
FC_TRACE=1 timeout -s KILL 600 python scripts/time_codec.py 256 64 2>&1 | grep "\[compress\]" | tail -13
timeout -s KILL 600 python scripts/time_codec.py 256 64 2>&1 | tail -6
