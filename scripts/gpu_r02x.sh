# round 2: int8 epilogue — mask-loop appends, refresh 32; tests + timing + ncu of the rescore
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02x_tests.log 2>&1; echo "i8 tests rc=$?" >> gpurun_out/r02x_tests.log
tail -3 gpurun_out/r02x_tests.log
run() { echo "== $*" >> gpurun_out/r02x.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -2 >> gpurun_out/r02x.log; }
ROWS=1000000
run FC_SHORTLIST_DEBUG=16
run FC_X=1
run FC_SHORTLIST_REFRESH=64
run FC_SHORTLIST_REFRESH=16
ROWS=125000
run FC_X=1
cat gpurun_out/r02x.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rescore_i8 -s 2 -c 1 -o gpurun_out/r02x_rescore python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02x_ncu.log 2>&1; echo "ncu rc=$?"
