timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shortlist_merge|k_rescore" -s 10 -c 2 -o gpurun_out/mr python bench.py --steps 3 --warmup 3 --no-cpu --no-codec --no-scoring --no-engine > gpurun_out/ncu_mr.log 2>&1
echo rc=$?
