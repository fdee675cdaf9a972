set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_i.err
python -c "import json; d=json.load(open('gpurun_out/bench_i.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['codec']['compress_GBps'], d['codec']['roofline']['frac'], d['engine']['requests_per_s'], d['clocks'])"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_shortlist_merge|k_rescore" -s 10 -c 2 -o gpurun_out/merge_rescore python bench.py --steps 3 --warmup 3 --no-cpu --no-codec --no-scoring --no-engine > gpurun_out/ncu_mr.log 2>&1; echo "ncu2 rc=$?"
