# round 2: engine A/B — HEAD vs device fix-up dot table (same flags, phase traces)
export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for D in _wt_old .; do
  echo "== $D"
  (cd $D && FC_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-codec --no-scoring --no-cpu --mixed-requests 4096 > /tmp/b.json 2> /tmp/b.err; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['engine']['requests_per_s'], d['engine']['mixed']['requests_per_s'])"; grep "^\[engine\]" /tmp/b.err | awk '{for(i=2;i<=NF;i+=2){s[$i]+=$(i+1)}} END{for(k in s) printf "%s %.1f ", k, s[k]; print ""}')
done; done
