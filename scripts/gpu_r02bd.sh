# round 2: ncu of K7 (k_inter_cert<5>) on config[4]
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_inter_cert -s 1 -c 1 -o gpurun_out/r02bd_k7 python scripts/time_codec.py 32 64 72x128x4 > gpurun_out/r02bd_ncu.log 2>&1; echo "ncu rc=$?"
