# round 2: units per worker (8 vs 16) at 1M / 250k / 125k rows on the tuned code
export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for R in 1000000 250000 125000; do for U in 16 8 12; do echo "== rows=$R UPW=$U"; FC_SHORTLIST_UPW=$U timeout -s KILL 300 python scripts/time_lookup.py $R 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/; s/fallback.*per step ms://'; done; done; done
