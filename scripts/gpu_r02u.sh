# round 2: int8 — contiguous per-query candidates + U-ordered rescore; tests then timing
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02u_tests.log 2>&1; echo "i8 tests rc=$?" >> gpurun_out/r02u_tests.log
tail -4 gpurun_out/r02u_tests.log
run() { echo "== $*" >> gpurun_out/r02u.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -2 >> gpurun_out/r02u.log; }
ROWS=1000000
run FC_SHORTLIST_DEBUG=16
run FC_X=1
run FC_LOOKUP_I8_PILOT=0
run FC_LOOKUP_I8_SLACK=0.002
ROWS=125000
run FC_X=1
cat gpurun_out/r02u.log
timeout -s KILL 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02u_tests2.log 2>&1; echo "lookup tests rc=$?" >> gpurun_out/r02u_tests2.log
tail -3 gpurun_out/r02u_tests2.log
