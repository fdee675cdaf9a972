export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-codec --no-scoring --no-engine > gpurun_out/r02cp_bench.json 2> gpurun_out/r02cp_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02cp_bench.json')); print(d['value'], d['cpu_baseline'])"; tail -2 gpurun_out/r02cp_bench.err
