# round 2: where the MMA warp waits (8 epilogue warps), with/without the filter, ring depth
export CUDA_MODULE_LOADING=EAGER
for rows in 1000000 125000; do
  for cfg in "16 6" "20 6" "16 5" "16 4" "18 6"; do
    set -- $cfg
    FC_SHORTLIST_DEBUG=$1 FC_SHORTLIST_NSTAGE=$2 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 | tr '\n' ' ' >> gpurun_out/r02n_sweep.log
    echo " <- dbg=$1 nstage=$2" >> gpurun_out/r02n_sweep.log
  done
done
