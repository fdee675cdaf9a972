# round 2: int8 main pass, one box per stage (16 stages) vs two (8) — timing without the debug counters
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/time_lookup.py $R 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/; s/fallback.*per step ms://'; }
for rep in 1 2; do
R=1000000; run FC_X=1; run FC_SHORTLIST_BPS=1; run FC_SHORTLIST_BPS=1 FC_SHORTLIST_MINCAP=48
done
R=125000; run FC_X=1; run FC_SHORTLIST_BPS=1
