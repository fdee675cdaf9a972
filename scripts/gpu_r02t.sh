# round 2: int8 pilot threshold (R-th best of the sample) — tests, then timing
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02t_tests.log 2>&1; echo "i8 tests rc=$?" >> gpurun_out/r02t_tests.log
tail -4 gpurun_out/r02t_tests.log
run() { echo "== $*" >> gpurun_out/r02t.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -2 >> gpurun_out/r02t.log; }
ROWS=1000000
run FC_SHORTLIST_DEBUG=16
run FC_X=1
run FC_LOOKUP_I8_SLACK=0.002
run FC_LOOKUP_I8_PILOT=0
ROWS=125000
run FC_X=1
run FC_LOOKUP_I8=0
cat gpurun_out/r02t.log
