export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/gram_r1b python scripts/time_codec.py 256 > gpurun_out/ncu_gram.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_gram.log
