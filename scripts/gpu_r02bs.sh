# round 2: ncu of the int8 main pass at 125k rows (per-rank size at 8 GPUs) with the debug cycle counters
export CUDA_MODULE_LOADING=EAGER
FC_SHORTLIST_DEBUG=16 timeout -s KILL 300 python scripts/time_lookup.py 125000 32 768 2>&1 | grep -E "stats|rows=" | head -4
FC_SHORTLIST_DEBUG=16 timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep -E "stats|rows=" | head -4
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k_shortlist_pair -s 3 -c 1 -o gpurun_out/r02bs_sl125k python scripts/time_lookup.py 125000 32 768 > gpurun_out/r02bs_ncu.log 2>&1; echo "ncu rc=$?"
