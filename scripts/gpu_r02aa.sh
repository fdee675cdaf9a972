# round 2: sort-free int8 rescore — tests + timing
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py tests/test_gpu_lookup.py -q -x > gpurun_out/r02aa_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02aa_tests.log
run() { echo "== $*" >> gpurun_out/r02aa.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02aa.log; }
ROWS=1000000
run FC_X=1
ROWS=125000
run FC_X=1
cat gpurun_out/r02aa.log
