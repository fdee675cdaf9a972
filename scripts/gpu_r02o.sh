# round 2 re-entry: full GPU suite + smoke + bench on the 8-warp-epilogue code
set -x
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02o_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r02o_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r02o_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02o_bench.json')); print(d['value'], d['e2e']['value'], d['roofline'], d.get('kernel_ms'), d['codec']['compress_GBps'], d['codec']['roofline']['frac'], d['engine']['requests_per_s'], d['clocks'])"
