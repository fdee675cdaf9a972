export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python -m pytest tests/test_gpu_store.py tests/test_capi.py -q -x -m gpu 2>&1 | tail -3
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-codec > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo rc=$?; tail -2 gpurun_out/bench_e.err
