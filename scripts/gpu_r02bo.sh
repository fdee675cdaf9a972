# round 2: NCCL communicator (world 1) through the sharded C-ABI + the sharded suite
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_sharded_capi.py -q -x > gpurun_out/r02bo_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r02bo_tests.log
