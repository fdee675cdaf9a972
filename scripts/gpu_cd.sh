export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_store.py -q -x -m gpu 2>&1 | tail -3
FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 2>&1 | tail -14
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"k_inter|k_gram_tc|k_pack_frames" -c 3 -o gpurun_out/prof_codec python scripts/time_codec.py 64 > gpurun_out/ncu_codec.log 2>&1; echo ncu rc=$?
