# round 2: fresh baseline of HEAD — lookup timing at 1M / 250k / 125k rows, full bench
export CUDA_MODULE_LOADING=EAGER
run() { echo "== rows=$ROWS $*" >> gpurun_out/r02af.log; env "$@" timeout -s KILL 180 python scripts/time_lookup.py $ROWS 32 768 2>&1 | tail -1 >> gpurun_out/r02af.log; }
for ROWS in 1000000 250000 125000; do run FC_X=1; done
cat gpurun_out/r02af.log
timeout -s KILL 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02af_bench.json 2> gpurun_out/r02af_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02af_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02af_bench.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['kernel_ms'], d['lookup_stats'], d['clocks']); print('codec', {k: d['codec'][k] for k in ('compress_GBps','compress_frac_hbm','decompress_GBps_e2e','decompress_frac_hbm_e2e')}); print('engine', d['engine'].get('requests_per_s'), d['engine'].get('index_stats'))"
