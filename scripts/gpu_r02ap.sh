# round 2: Gram with two MMAs per K step (HH, HL; HL^T added by select)
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep -E "select:|K7 cert|gram \+ select" | head -4
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_capi.py -q -x -m gpu > gpurun_out/r02ap_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ap_tests.log
FC_COMPRESS_SPLIT=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/r02ap_gram python scripts/time_codec.py 256 > gpurun_out/r02ap_ncu.log 2>&1; echo "ncu rc=$?"
