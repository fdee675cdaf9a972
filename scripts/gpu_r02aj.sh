# round 2: rescore prefetch variants (bit0 prescore window, bit1 exact bulk prefetch, bit2 early fp32 prefetch) x blocks/SM
export CUDA_MODULE_LOADING=EAGER
run() { echo "== rows=$ROWS $*" >> gpurun_out/r02aj.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 | sed 's/.*rescore /rescore /; s/, shortlist_tier2.*//' >> gpurun_out/r02aj.log; }
for ROWS in 1000000 125000; do for F in 0 1 2 3 7; do for B in 3 4; do run FC_RI_MINB=$B FC_RI_FLAGS=$F; done; done; done
cat gpurun_out/r02aj.log
