# round 2: scoring phase breakdown with a stamp after the survivor load
export CUDA_MODULE_LOADING=EAGER
FC_SCORE_PHASES=1 timeout -s KILL 600 python scripts/time_store.py 100000 gets 2>&1 | grep "score phases\|raw:" | tail -2
