export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_lookup.py tests/test_engine.py -q -x -k "not large" > gpurun_out/san3.log 2>&1; echo "san3 rc=$?"; tail -6 gpurun_out/san3.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_lookup.py -q -x -k "near_tied" > gpurun_out/san4.log 2>&1; echo "san4 rc=$?"; tail -6 gpurun_out/san4.log
