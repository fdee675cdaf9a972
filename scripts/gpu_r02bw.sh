# round 2: compress part split for 16+ prompts (config[4] batches of 32 now take two parts)
export CUDA_MODULE_LOADING=EAGER
for S in 1 2; do echo "config4 split $S"; FC_COMPRESS_SPLIT=$S timeout -s KILL 300 python scripts/time_codec.py 32 64 72x128x4 2>&1 | head -3; done
echo "config2 default"; timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
