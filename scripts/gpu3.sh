python __graft_entry__.py 2>&1 | tail -5
timeout -s KILL 300 python -m pytest tests/test_gpu_store.py -q -m gpu -k hole 2>&1 | tail -5
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
