# round 2: ncu (source counters) of the int8 main pass after the pilot / refresh changes
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_shortlist_pair -s 3 -c 1 -o gpurun_out/r02cf_main python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02cf_ncu.log 2>&1; echo "ncu rc=$?"
FC_SHORTLIST_DEBUG=16 timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep stats | head -2
