# round 2: scoring kernel timing (kernel-only timer) + ncu of k_policy_fused
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | tail -5
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_policy_fused -s 3 -c 1 -o gpurun_out/r02bk_policy python scripts/time_store.py 100000 gets > gpurun_out/r02bk_ncu.log 2>&1; echo "ncu rc=$?"
