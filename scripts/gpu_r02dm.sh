# round 2: single-GPU proxy for the cross-rank pilot-key exchange at the G = 8 shard size (125k rows):
# a pilot over every 2nd tile is the sample 8 ranks' every-16th-tile pilots give together
export CUDA_MODULE_LOADING=EAGER
for s in 16 2; do echo "stride $s"; FC_LOOKUP_I8_PILOT_STRIDE=$s timeout -s KILL 300 python scripts/time_lookup.py 125000 32 768 2>&1 | tail -1; done
