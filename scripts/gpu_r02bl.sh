# round 2: fused scoring with register-resident keys — timing (REG on/off), store tests, ncu
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | tail -2
FC_SCORE_REG=0 timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | tail -1
timeout -s KILL 1500 python -m pytest tests/test_gpu_store.py tests/test_gpu_snapshot.py tests/test_engine.py -q -x -m gpu > gpurun_out/r02bl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02bl_tests.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_policy_fused -s 3 -c 1 -o gpurun_out/r02bl_policy python scripts/time_store.py 100000 gets > gpurun_out/r02bl_ncu.log 2>&1; echo "ncu rc=$?"
