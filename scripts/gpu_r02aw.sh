export CUDA_MODULE_LOADING=EAGER
nproc; python -c "import os; print(os.cpu_count(), len(os.sched_getaffinity(0)))"
FC_COMPRESS_SPLIT=1 FC_TRACE=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | grep -E "^\[compress\]|^compress" | tail -16
