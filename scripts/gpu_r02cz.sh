# round 2: int8 tier candidate list sizes on the tuned code (kout merged per query, kunit per unit list)
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1 | sed 's/, shortlist_tier2/ | tier2/; s/rows=.*: step/step/; s/, rescore_tier2.*//'; }
run FC_X=1
run FC_LOOKUP_I8_KOUT=224
run FC_LOOKUP_I8_KOUT=192
run FC_LOOKUP_I8_KUNIT=24
run FC_LOOKUP_I8_KUNIT=16
run FC_LOOKUP_I8_KUNIT=48
