# round 2: Gram pass pipeline depth sweep (fp32 smem stages NX, L2 prefetch distance PF)
export CUDA_MODULE_LOADING=EAGER
for C in 4,8 4,4 4,2 4,0 5,4 3,4; do echo "== NX,PF=$C"; FC_GRAM_CFG=$C FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 2,3p; done
