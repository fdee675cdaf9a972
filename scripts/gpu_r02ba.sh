# round 2: compress A/B — HEAD (two halves, each Gram+select+assembly) vs whole-batch Gram/select + staged assembly parts
export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do
echo "old split2"; (cd _wt_old && FC_COMPRESS_SPLIT=2 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3)
for S in 2 3 4; do echo "new split $S"; FC_COMPRESS_SPLIT=$S timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3; done
done
