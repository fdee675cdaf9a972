# round 2: full bench repeat (engine regression check), HEAD then 8de5b56
export CUDA_MODULE_LOADING=EAGER
for D in . _wt_old; do
(cd $D && timeout -s KILL 1500 python bench.py --steps 20 --warmup 5 --no-cpu > /tmp/b.json 2> /tmp/b.err; python -c "import json; d=json.load(open('/tmp/b.json')); print('$D', d['value'], d['engine'].get('requests_per_s'), d['engine']['mixed']['requests_per_s'], d['codec']['compress_frac_hbm'], d['codec']['decompress_frac_hbm_e2e'])")
done
