# round 2: int8 rescore, 3 chunks per lane at dim <= 768: 5 blocks/SM (96 regs, small spill) vs 4
export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for B in 5 4; do echo "== MINB=$B"; FC_RI_MINB=$B timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/; s/fallback.*per step ms://'; done; done
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py -q -x > gpurun_out/r02cl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02cl_tests.log
