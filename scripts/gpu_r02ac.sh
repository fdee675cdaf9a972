# round 2: threshold tier tests (rest of the file) + units-per-worker sweep at 125k / 1M
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02ac_tests.log 2>&1; echo "tests rc=$?"; grep -E "clustered vs plain|passed|failed|Error" gpurun_out/r02ac_tests.log | tail -8
run() { echo "== $*" >> gpurun_out/r02ac.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02ac.log; }
ROWS=125000
run FC_SHORTLIST_UPW=16
run FC_SHORTLIST_UPW=8
run FC_SHORTLIST_UPW=4
run FC_SHORTLIST_UPW=2
ROWS=1000000
run FC_SHORTLIST_UPW=8
run FC_SHORTLIST_UPW=4
cat gpurun_out/r02ac.log
