# round 2: config[3] at its stated size (100k requests) + parity prefix vs the serial restatement
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 600 python scripts/config3_scale.py --requests 2048 --capacity-gb 2 --prefix 64 --prefix-capacity-gb 0.1 > gpurun_out/r02au_small.json 2> gpurun_out/r02au_small.err; echo "small rc=$?"; tail -c 1500 gpurun_out/r02au_small.json; tail -3 gpurun_out/r02au_small.err
timeout -s KILL 1800 python scripts/config3_scale.py > gpurun_out/r02au_config3.json 2> gpurun_out/r02au_config3.err; echo "full rc=$?"; cat gpurun_out/r02au_config3.json; tail -3 gpurun_out/r02au_config3.err
