timeout -s KILL 900 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_h.err
python -c "import json; d=json.load(open('gpurun_out/bench_h.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['ms_per_step_median'], d['clocks'])"
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/r01c_shortlist_pair python scripts/time_lookup.py 1000000 32 768 > gpurun_out/ncu_sl.log 2>&1; echo ncu=$?
