# round 2: int8 rescore — size of the first pre-scored set A (32 default)
export CUDA_MODULE_LOADING=EAGER
for A in 32 16 24 48 64; do echo "== A=$A"; FC_RI_A=$A timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/'; done
