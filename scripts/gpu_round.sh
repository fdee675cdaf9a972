set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_i.err
python -c "import json; d=json.load(open('gpurun_out/bench_i.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['frac'], d['codec']['compress_GBps'], d['codec']['roofline']['frac'], d['engine']['requests_per_s'], d['clocks'])"
