# round 2: ncu of the Gram pass (one part) with source counters
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/r02al_gram python scripts/time_codec.py 256 > gpurun_out/r02al_ncu.log 2>&1; echo "ncu rc=$?"
