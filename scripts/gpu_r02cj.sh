# round 2: ncu of the int8 pilot launch (every 16th row tile) with the debug cycle counters
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/r02cj_pilot python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02cj_ncu.log 2>&1; echo "ncu rc=$?"
