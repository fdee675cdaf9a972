# round 2: rescore — early fp32 prefetch, 16-deep exact loads, 3 vs 4 blocks/SM
export CUDA_MODULE_LOADING=EAGER
run() { echo "== rows=$ROWS $*" >> gpurun_out/r02ai.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02ai.log; }
for ROWS in 1000000 125000; do run FC_RI_MINB=4; run FC_RI_MINB=3; done
cat gpurun_out/r02ai.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rescore_i8 -s 2 -c 1 -o gpurun_out/r02ai_rescore python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02ai_ncu.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py -q -x > gpurun_out/r02ai_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ai_tests.log
