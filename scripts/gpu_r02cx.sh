# round 2: int8 threshold slack (hoff = typical eps + slack) on the tuned code
export CUDA_MODULE_LOADING=EAGER
for S in 0.003 0.002 0.001 0.0 0.005; do echo "== slack=$S"; FC_LOOKUP_I8_SLACK=$S timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2/ | tier2/; s/rows=.*: step/step/'; done
