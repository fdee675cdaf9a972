export CUDA_MODULE_LOADING=EAGER FC_LOOKUP_DIAG=1
for cta in 2 1; do for d in 0 1 2 4 6; do echo "cta=$cta debug=$d"; FC_SHORTLIST_CTA=$cta FC_SHORTLIST_DEBUG=$d timeout -s KILL 120 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1; done; done
