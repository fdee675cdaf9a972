set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c.err
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-engine > gpurun_out/ncu_c.log 2>&1; echo c=$?
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_gram_tc|k_inter_cert|k_pack_frames" -c 3 -o gpurun_out/r01b_codec python scripts/time_codec.py 256 > gpurun_out/ncu_b.log 2>&1; echo b=$?
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"k_policy" -c 5 -o gpurun_out/r01b_policy python scripts/time_store.py 100000 > gpurun_out/ncu_p.log 2>&1; echo p=$?
