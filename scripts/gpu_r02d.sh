# round 2: packed shortlist candidates (fp16 round-up score | row offset) +
# deeper TMA ring; sharded C-ABI; parity suites
export CUDA_MODULE_LOADING=EAGER
timeout 1200 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py tests/test_gpu_sharded_capi.py tests/test_capi.py tests/test_engine.py -x -q > gpurun_out/r02d_tests.log 2>&1; echo rc=$? >> gpurun_out/r02d_tests.log
for rows in 1000000 125000; do
  FC_SHORTLIST_DEBUG=16 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 >> gpurun_out/r02d_time.log
  timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -1 >> gpurun_out/r02d_time.log
done
