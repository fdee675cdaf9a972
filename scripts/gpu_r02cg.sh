# round 2: int8 main pass table ring: boxes per stage x candidate-list floor (more stages)
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" FC_SHORTLIST_DEBUG=16 timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep -E "stats|rows=" | tail -2 | sed 's/, shortlist_tier2.*//; s/rows=.*: step/step/; s/fallback.*per step ms://; s/shortlist.i8. stats: warp-tiles [0-9]* //'; }
run FC_X=1
run FC_SHORTLIST_MINCAP=48
run FC_SHORTLIST_MINCAP=40
run FC_SHORTLIST_BPS=3
run FC_SHORTLIST_BPS=3 FC_SHORTLIST_MINCAP=40
run FC_SHORTLIST_BPS=1
