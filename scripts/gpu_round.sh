set -x
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_f.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
