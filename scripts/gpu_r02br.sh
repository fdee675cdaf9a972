# round 2: small-shard (125k rows, the 8-GPU per-rank size) shortlist knobs: histogram refresh interval x units per worker
export CUDA_MODULE_LOADING=EAGER
for RF in 64 16 8 4; do for U in 16 8; do echo "== REFRESH=$RF UPW=$U"; FC_SHORTLIST_REFRESH=$RF FC_SHORTLIST_UPW=$U timeout -s KILL 300 python scripts/time_lookup.py 125000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//'; done; done
for RF in 64 32; do echo "== 1M REFRESH=$RF"; FC_SHORTLIST_REFRESH=$RF timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//'; done
