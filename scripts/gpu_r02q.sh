# round 2: int8 tier-1 lookup — parity tests first, then timing i8 vs bf16
export CUDA_MODULE_LOADING=EAGER PYTHONFAULTHANDLER=1
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup_i8.py -q -x -s > gpurun_out/r02q_i8_tests.log 2>&1; echo "i8 tests rc=$?" >> gpurun_out/r02q_i8_tests.log
tail -15 gpurun_out/r02q_i8_tests.log
for rows in 1000000 125000; do
  FC_SHORTLIST_DEBUG=16 timeout -s KILL 180 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -3 >> gpurun_out/r02q_time.log
  timeout -s KILL 180 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -1 >> gpurun_out/r02q_time.log
  FC_LOOKUP_I8=0 timeout -s KILL 180 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -1 >> gpurun_out/r02q_time.log
done
cat gpurun_out/r02q_time.log
timeout -s KILL 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02q_tests.log 2>&1; echo "lookup tests rc=$?" >> gpurun_out/r02q_tests.log
tail -5 gpurun_out/r02q_tests.log
