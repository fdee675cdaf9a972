timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_g.err
python -c "import json; d=json.load(open('gpurun_out/bench_g.json')); c=d['codec']; print(d['value'], c['compress_GBps'], c['compress_s_reps'], d['lookup_stats'])"
