# round 2: compress host timeline, one part (FC_COMPRESS_SPLIT=1) and two parts, config[2] batch
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 600 python scripts/time_codec.py 256 64 > gpurun_out/r02di_split1.log 2>&1
FC_TRACE=1 timeout -s KILL 600 python scripts/time_codec.py 256 64 > gpurun_out/r02di_split2.log 2>&1
grep "\[compress\]" gpurun_out/r02di_split1.log | tail -14; grep "wall" gpurun_out/r02di_split1.log
