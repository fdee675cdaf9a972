# round 2: sort-free rescore (threshold sets by bisection, L2 bulk prefetch, fp64 query in smem)
export CUDA_MODULE_LOADING=EAGER
run() { echo "== rows=$ROWS $*" >> gpurun_out/r02ag.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02ag.log; }
for ROWS in 1000000 125000; do run FC_X=1; done
cat gpurun_out/r02ag.log
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py tests/test_gpu_sharded_capi.py -q -x > gpurun_out/r02ag_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ag_tests.log
