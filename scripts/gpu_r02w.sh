# round 2: int8 kernel with 3 accumulator buffers (A partly in smem) — tests + timing
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02w_tests.log 2>&1; echo "i8 tests rc=$?" >> gpurun_out/r02w_tests.log
tail -3 gpurun_out/r02w_tests.log
run() { echo "== $*" >> gpurun_out/r02w.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -2 >> gpurun_out/r02w.log; }
ROWS=1000000
run FC_SHORTLIST_DEBUG=16
run FC_X=1
run FC_SHORTLIST_NSTAGE=6
run FC_SHORTLIST_BPS=1
ROWS=125000
run FC_X=1
cat gpurun_out/r02w.log
