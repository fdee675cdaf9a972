# round 2: compress phase trace (one part and two parts)
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 > gpurun_out/r02ak_split1.log 2>&1
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 > gpurun_out/r02ak_split1_trace.log 2>&1
timeout -s KILL 300 python scripts/time_codec.py 256 > gpurun_out/r02ak_split2.log 2>&1
grep -v "^\[compress\]" gpurun_out/r02ak_split1.log | head; tail -30 gpurun_out/r02ak_split1_trace.log; cat gpurun_out/r02ak_split2.log | head -5
