timeout -s KILL 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py -q -x -k "not codec" 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-codec --no-scoring --no-engine > gpurun_out/bench_lk.json 2>gpurun_out/bench_lk.err; python -c "import json; d=json.load(open('gpurun_out/bench_lk.json')); print(d['value'], d['ms_per_step_median'], d['ms_per_step_max'], d['kernel_ms'])"; done
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_shortlist_merge|k_rescore" -c 4 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep -E "k_shortlist_merge|k_rescore|gpu__time_duration" | head -8
