# round 2: lookup diagnostics (debug-flag timings at 1M and 125k rows), the
# new parity tests, and one ncu --set full capture of the shortlist kernel
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02a_tests.log 2>&1; echo tests=$?
for rows in 1000000 125000; do
  for dbg in 0 4 32 1 2 3 16; do
    FC_SHORTLIST_DEBUG=$dbg FC_LOOKUP_DIAG=$([ $dbg = 0 ] && echo 0 || echo 1) timeout 120 python scripts/time_lookup.py $rows 32 768 >> gpurun_out/r02a_dbg.log 2>&1
    echo "  ^ dbg=$dbg" >> gpurun_out/r02a_dbg.log
  done
done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/r02a_shortlist python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02a_ncu.log 2>&1; echo ncu=$?
