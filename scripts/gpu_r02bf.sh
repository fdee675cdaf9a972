# round 2: config[4] per GPU through the engine (72x128x4 latents, evicting budget, periodic whole-cache checkpoints) + parity prefix
export CUDA_MODULE_LOADING=EAGER
df -h /dev/shm | tail -1; free -g | head -2
timeout -s KILL 600 python scripts/config3_scale.py --dims 72x128x4 --batch 64 --requests 512 --capacity-gb 2 --checkpoint-every 256 --prefix 48 --prefix-capacity-gb 0.5 > gpurun_out/r02bf_small.json 2> gpurun_out/r02bf_small.err; echo "small rc=$?"; cat gpurun_out/r02bf_small.json; tail -3 gpurun_out/r02bf_small.err
timeout -s KILL 2400 python scripts/config3_scale.py --dims 72x128x4 --batch 64 --requests 25000 --capacity-gb 16 --checkpoint-every 5000 --prefix 96 --prefix-capacity-gb 1 > gpurun_out/r02bf_config4.json 2> gpurun_out/r02bf_config4.err; echo "full rc=$?"; cat gpurun_out/r02bf_config4.json; tail -3 gpurun_out/r02bf_config4.err
