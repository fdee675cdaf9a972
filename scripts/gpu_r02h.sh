# round 2: pipelined TMEM loads + popc appends in the shortlist epilogue; sharded-store fix
export CUDA_MODULE_LOADING=EAGER PYTHONFAULTHANDLER=1
for rows in 1000000 125000; do
  FC_SHORTLIST_DEBUG=16 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 >> gpurun_out/r02h_time.log
  timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -1 >> gpurun_out/r02h_time.log
done
timeout 300 tests/cpp/_build/sharded_kat > gpurun_out/r02h_kat.log 2>&1; echo kat=$? >> gpurun_out/r02h_kat.log
timeout 1200 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_sharded_capi.py tests/test_gpu_snapshot.py tests/test_engine.py tests/test_capi.py -q -x > gpurun_out/r02h_tests.log 2>&1; echo rc=$? >> gpurun_out/r02h_tests.log
