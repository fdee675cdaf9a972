# round 2: engine fix-up dots from one device table per batch; engine tests + engine bench sections with phase traces
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_engine.py tests/test_cli.py -q -x -m gpu > gpurun_out/r02bu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02bu_tests.log
FC_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-codec --no-scoring --no-cpu > /tmp/b.json 2> /tmp/b.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['engine']['requests_per_s'], d['engine']['mixed']['requests_per_s'])"; grep "^\[engine\]" /tmp/b.err | awk '{for(i=2;i<=NF;i+=2){s[$i]+=$(i+1)}} END{for(k in s) printf "%s %.1f ", k, s[k]; print ""}'
