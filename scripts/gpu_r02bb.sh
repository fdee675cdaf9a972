# round 2: config[4] codec breakdown (32 prompts x 5 x 64 x 72x128x4)
export CUDA_MODULE_LOADING=EAGER
for S in 1 2; do echo "split $S"; FC_COMPRESS_SPLIT=$S timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | head -4; done
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | grep "^\[compress\]" | tail -13
