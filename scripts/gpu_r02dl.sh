# round 2: full GPU suite + smoke + full bench (final validation of the round-2 build)
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02dl_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02dl_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02dl_bench.json 2> gpurun_out/r02dl_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02dl_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02dl_bench.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['clocks']); print('codec', {k: d['codec'][k] for k in ('compress_GBps','compress_frac_hbm','decompress_GBps_e2e','decompress_frac_hbm_e2e')}, d['codec']['roofline']); print('large', {k: d['codec_large'][k] for k in ('compress_frac_hbm','decompress_frac_hbm_e2e')}, d['codec_large']['checkpoint']['save_GBps']); print('scoring', d['scoring'].get('scoring_ms_per_launch')); print('engine', d['engine'].get('requests_per_s'), d['engine']['mixed']['requests_per_s'])"
