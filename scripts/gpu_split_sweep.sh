export CUDA_MODULE_LOADING=EAGER
for S in 1 2 3 4 6; do echo "split $S"; FC_COMPRESS_SPLIT=$S timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 3p; done
