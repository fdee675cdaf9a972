# round 2: codec bench with the stream-ordered decompress (timing sync fixed)
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-scoring --no-engine --no-cpu > gpurun_out/r02an_bench.json 2> gpurun_out/r02an_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r02an_bench.err
python -c "import json; d=json.load(open('gpurun_out/r02an_bench.json')); print(d['value']); print('codec', {k: d['codec'][k] for k in ('compress_GBps','compress_frac_hbm','decompress_GBps_e2e','decompress_frac_hbm_e2e')}, d['codec']['roofline']); print('large', {k: d['codec_large'][k] for k in ('compress_frac_hbm','decompress_frac_hbm_e2e')})"
