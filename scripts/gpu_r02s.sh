# round 2: int8 shortlist — timing with prefetched tile scales + lazy keys, then one ncu capture with source
export CUDA_MODULE_LOADING=EAGER FC_LOOKUP_I8_SLACK=0.003
run() { echo "== $*" >> gpurun_out/r02s.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -2 >> gpurun_out/r02s.log; }
run FC_SHORTLIST_DEBUG=16
run FC_X=1
run FC_LOOKUP_I8=0
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/r02s_i8 python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02s_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r02s.log
cat gpurun_out/r02s.log
