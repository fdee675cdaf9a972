export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-scoring --no-engine --no-cpu > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02bh_bench.json')); print(d['codec_large']['checkpoint'], d['codec']['compress_frac_hbm'])"
