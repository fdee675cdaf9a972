# round 2 (final build): config[3] at stated size and config[4] per GPU, each with its parity prefix vs the serial restatement
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1800 python scripts/config3_scale.py > gpurun_out/r02dj_config3.json 2> gpurun_out/r02dj_config3.err; echo "config3 rc=$?"; tail -c 1200 gpurun_out/r02dj_config3.json; tail -2 gpurun_out/r02dj_config3.err
timeout -s KILL 2400 python scripts/config3_scale.py --dims 72x128x4 --batch 64 --requests 25000 --capacity-gb 16 --checkpoint-every 5000 --prefix 96 --prefix-capacity-gb 1 > gpurun_out/r02dj_config4.json 2> gpurun_out/r02dj_config4.err; echo "config4 rc=$?"; tail -c 1500 gpurun_out/r02dj_config4.json; tail -2 gpurun_out/r02dj_config4.err
