timeout -s KILL 200 python -m pytest -q -x tests/test_gpu_lookup.py -m gpu 2>&1 | tail -2
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_shortlist -s 2 -c 1 -o gpurun_out/prof_shortlist python scripts/time_lookup.py 1000000 64 > gpurun_out/ncu1.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu1.log
