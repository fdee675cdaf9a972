# round 2: int8 — pilot units, prescore count; store fused scoring tests + timing; ncu of the main int8 pass
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*" >> gpurun_out/r02v.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02v.log; }
ROWS=1000000
run FC_X=1
run FC_X=2
ROWS=125000
run FC_X=1
cat gpurun_out/r02v.log
timeout -s KILL 900 python -m pytest tests/test_gpu_store.py -q -x > gpurun_out/r02v_store.log 2>&1; echo "store tests rc=$?" >> gpurun_out/r02v_store.log
tail -3 gpurun_out/r02v_store.log
timeout -s KILL 300 python scripts/time_store.py 100000 gets > gpurun_out/r02v_store_time.log 2>&1
FC_SCORE_FUSED=0 timeout -s KILL 300 python scripts/time_store.py 100000 gets >> gpurun_out/r02v_store_time.log 2>&1
cat gpurun_out/r02v_store_time.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_shortlist_pair -s 3 -c 1 -o gpurun_out/r02v_i8main python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02v_ncu.log 2>&1; echo "ncu rc=$?"
