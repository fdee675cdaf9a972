export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_shortlist_pair -s 2 -c 1 -o gpurun_out/r01_shortlist_pair python scripts/time_lookup.py 1000000 32 768 > gpurun_out/ncu_a.log 2>&1; echo a=$?
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"k_decompress$|k_gram_tc|k_inter|k_pack_frames|k_decompress_stitch" -c 5 -o gpurun_out/r01_codec python scripts/time_codec.py 256 > gpurun_out/ncu_b.log 2>&1; echo b=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-scoring > gpurun_out/ncu_c.log 2>&1; echo c=$?
