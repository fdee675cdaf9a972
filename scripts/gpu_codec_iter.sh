# round 2: compress iteration — timing (1 part, trace, 2 parts), codec parity tests, ncu of k_gram_tc. usage: bash scripts/gpu_codec_iter.sh TAG [ncu]
export CUDA_MODULE_LOADING=EAGER
T=$1
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep -E "select:|K7 cert" | head -2
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | head -3
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_capi.py -q -x -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
if [ "$2" = ncu ]; then FC_COMPRESS_SPLIT=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/${T}_gram python scripts/time_codec.py 256 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"; fi
