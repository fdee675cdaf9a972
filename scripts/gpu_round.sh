set -x
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_e.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-engine > gpurun_out/ncu_c.log 2>&1; echo c=$?
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"k_policy" -c 7 -o gpurun_out/r01c_policy python scripts/time_store.py 100000 gets > gpurun_out/ncu_p.log 2>&1; echo p=$?
