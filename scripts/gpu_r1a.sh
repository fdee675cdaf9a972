set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cat MEASURED_PEAKS.json 2>/dev/null; ls /root/repo/MEASURED_PEAKS.json 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout -s KILL 300 python __graft_entry__.py 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_a.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -3 gpurun_out/bench_ref.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo "ncu-launch rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_shortlist2 -s 2 -c 1 -o gpurun_out/prof_shortlist2 python scripts/time_lookup.py 1000000 32 768 > gpurun_out/ncu_sl.log 2>&1; echo ncu rc=$?
