FC_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-cpu --no-scoring --no-engine > gpurun_out/bench_g.json 2>gpurun_out/bench_g.err
grep "^\[compress\]" gpurun_out/bench_g.err | tail -30
