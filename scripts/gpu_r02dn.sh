# round 2 (final build): 20 minutes of randomized lookup/codec parity fuzzing against the oracle
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python scripts/fuzz_parity.py --minutes 20 --seed 29 > gpurun_out/r02dn_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -4 gpurun_out/r02dn_fuzz.log
