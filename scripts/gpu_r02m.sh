export CUDA_MODULE_LOADING=EAGER PYTHONFAULTHANDLER=1
for rows in 1000000 125000; do
  FC_SHORTLIST_DEBUG=16 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 >> gpurun_out/r02m_time.log
  timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -1 >> gpurun_out/r02m_time.log
done
timeout 900 python -m pytest tests/test_gpu_lookup.py -q -x > gpurun_out/r02m_tests.log 2>&1; echo rc=$? >> gpurun_out/r02m_tests.log
