# round 2: k_i8_merge two-level selection (score bucket, then the bucket's keys); rescore CPL=3; timing + lookup tests
export CUDA_MODULE_LOADING=EAGER
for R in 1000000 1000000 125000; do timeout -s KILL 300 python scripts/time_lookup.py $R 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//'; done
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py tests/test_gpu_fullsize.py tests/test_gpu_lookup.py tests/test_gpu_sharded_capi.py -q -x > gpurun_out/r02cm_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02cm_tests.log
