# round 2: randomized parity fuzzing on the current code (lookup int8 rescore, Gram/K7 changes)
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 720 python scripts/fuzz_parity.py --minutes 10 --seed 23 > gpurun_out/r02cu_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -5 gpurun_out/r02cu_fuzz.log
