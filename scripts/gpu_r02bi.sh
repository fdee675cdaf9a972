# round 2: ncu captures for the bench roofline traffic fields + launch list of the bench
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_shortlist_pair -s 3 -c 1 -o gpurun_out/r02bi_shortlist python scripts/time_lookup.py 1000000 32 768 > gpurun_out/r02bi_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k_decompress_groups -s 6 -c 1 -o gpurun_out/r02bi_decompress python scripts/time_codec.py 256 > gpurun_out/r02bi_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02bi_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-engine --no-large --no-scoring > gpurun_out/r02bi_b.log 2>&1; echo "launch list rc=$?"
