# round 2: packed-candidate shortlist, ring depth vs candidate-buffer depth
export CUDA_MODULE_LOADING=EAGER
for rows in 1000000 125000; do
  for cfg in "8 999" "7 999" "6 999" "6 256" "5 999"; do
    set -- $cfg
    FC_SHORTLIST_NSTAGE=$1 FC_SHORTLIST_CAPMAX=$2 FC_SHORTLIST_DEBUG=16 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 | tr '\n' ' ' >> gpurun_out/r02f_sweep.log
    echo " <- nstage=$1 capmax=$2" >> gpurun_out/r02f_sweep.log
  done
done
