# round 2: shortlist pipeline sweep (stages / boxes per stage / histogram refresh period)
export CUDA_MODULE_LOADING=EAGER
for rows in 1000000 125000; do
  for cfg in "6 2 16" "4 2 16" "3 2 16" "8 1 16" "6 1 16" "4 2 8" "4 2 4" "3 2 8" "2 2 16"; do
    set -- $cfg
    FC_SHORTLIST_NSTAGE=$1 FC_SHORTLIST_BPS=$2 FC_SHORTLIST_REFRESH=$3 FC_SHORTLIST_DEBUG=16 FC_LOOKUP_DIAG=1 timeout 120 python scripts/time_lookup.py $rows 32 768 2>&1 | tail -2 | tr '\n' ' ' >> gpurun_out/r02b_sweep.log
    echo " <- nstage=$1 bps=$2 refresh=$3" >> gpurun_out/r02b_sweep.log
  done
done
