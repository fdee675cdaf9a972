# round 2: ncu of the sort-free rescore
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rescore_i8 -s 2 -c 1 -o gpurun_out/r02ah_rescore python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02ah_ncu.log 2>&1; echo "ncu rc=$?"
