# round 2: main-pass histogram refresh interval at 1M rows (64 default) and 125k
export CUDA_MODULE_LOADING=EAGER
for RF in 64 128 256; do echo "== 1M REFRESH=$RF"; FC_SHORTLIST_REFRESH=$RF timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/'; done
for RF in 64 128; do echo "== 125k REFRESH=$RF"; FC_SHORTLIST_REFRESH=$RF timeout -s KILL 300 python scripts/time_lookup.py 125000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/'; done
