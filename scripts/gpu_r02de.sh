# round 2: scoring with a warp-shuffle block_pick and a rank-counting head sort — store/engine tests + phase breakdown
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1200 python -m pytest tests/test_gpu_store.py tests/test_engine.py tests/test_gpu_sharded_capi.py -q -x -k "not lookup_two_ranks" > gpurun_out/r02de_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02de_tests.log
FC_SCORE_PHASES=1 timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | grep "score phases\|raw:" | tail -2
