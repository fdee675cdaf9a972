# round 2: fused scoring phase breakdown (CTA-0 globaltimer stamps), 500k live steps, bench access pattern
export CUDA_MODULE_LOADING=EAGER
FC_SCORE_PHASES=1 timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | grep "score phases" | tail -2
FC_TRACE=1 timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | grep "score fused" | sort | uniq -c | sort -rn | head -5
