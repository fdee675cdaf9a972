export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_lookup.py -q -x -m gpu 2>&1 | tail -2
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo rc=$?; tail -2 gpurun_out/bench_d.err
