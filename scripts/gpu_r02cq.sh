export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-scoring --no-engine --no-large > gpurun_out/r02cq_bench.json 2> gpurun_out/r02cq_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02cq_bench.json')); print(d['cpu_baseline']['parity'], d['codec']['cpu_baseline'])"; tail -2 gpurun_out/r02cq_bench.err
