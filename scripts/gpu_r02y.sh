# round 2: int8 lookup (pilot mask-loop, refresh 64, rescore 6 blocks/SM) — timing, full GPU suite, smoke, bench
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*" >> gpurun_out/r02y.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02y.log; }
ROWS=1000000
run FC_X=1
ROWS=125000
run FC_X=1
cat gpurun_out/r02y.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02y_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02y_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02y_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02y_bench.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['kernel_ms'], d['lookup_stats'], d['clocks']); print('codec', {k: d['codec'][k] for k in ('compress_GBps','compress_frac_hbm','decompress_GBps_e2e','decompress_frac_hbm_e2e')}); print('large', d.get('codec_large')); print('scoring', d['scoring'].get('scoring_ms_per_launch'), d['scoring'].get('scoring_ms_per_call'), d['scoring'].get('evictions_per_s')); print('engine', d['engine'].get('requests_per_s'))"
