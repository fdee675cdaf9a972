export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 300 python -m pytest tests/test_gpu_lookup.py -q -x -m gpu 2>&1 | tail -3
timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768
FC_SHORTLIST_DEBUG=16 timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -2
FC_LOOKUP_DIAG=1 FC_SHORTLIST_DEBUG=4 timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/prof_pair2 python scripts/time_lookup.py 1000000 32 768 > gpurun_out/ncu_pair.log 2>&1; echo ncu rc=$?
