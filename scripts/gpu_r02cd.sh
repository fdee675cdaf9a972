export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for RF in 64 256 512 4096; do echo "== 1M REFRESH=$RF"; FC_SHORTLIST_REFRESH=$RF timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/; s/fallback.*per step ms://'; done; done
