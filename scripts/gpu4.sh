timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; tail -3 gpurun_out/bench2.err
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_shortlist2 -s 2 -c 1 -o gpurun_out/prof_shortlist2 python scripts/time_lookup.py 1000000 32 768 > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
