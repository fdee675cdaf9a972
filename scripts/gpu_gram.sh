for k in 1 2 6; do
  export FC_GRAM_KSPLIT=$k
  timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-cpu --no-scoring --no-engine > gpurun_out/bench_g.json 2>gpurun_out/bench_g.err
  python -c "import json; d=json.load(open('gpurun_out/bench_g.json')); c=d['codec']; print('ks=$k', c['compress_s_reps'], c['compress_kernel_ms'])"
done
