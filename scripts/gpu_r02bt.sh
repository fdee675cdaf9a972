# round 2: pilot sampling stride sweep at small shards (125k / 250k rows) and 1M
export CUDA_MODULE_LOADING=EAGER
for R in 125000 250000; do for S in 16 8 4 2; do echo "== rows=$R stride=$S"; FC_LOOKUP_I8_PILOT_STRIDE=$S timeout -s KILL 300 python scripts/time_lookup.py $R 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/'; done; done
for S in 16 8; do echo "== rows=1M stride=$S"; FC_LOOKUP_I8_PILOT_STRIDE=$S timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/'; done
