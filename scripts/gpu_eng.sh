for i in 1 2 3; do
FC_TRACE=1 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --rows 100000 --no-cpu --no-codec --no-scoring > gpurun_out/bench_eng.json 2>gpurun_out/bench_eng.err
python - <<'PY'
import json,re
d=json.load(open('gpurun_out/bench_eng.json')); e=d['engine']
lines=open('gpurun_out/bench_eng.err').read().splitlines()
print(round(e['requests_per_s']))
for l in lines:
    m=re.search(r'([0-9.]+) ms$', l)
    if m and float(m.group(1)) > 4 and not l.startswith('[engine]'): print(l)
    if l.startswith('[engine]'):
        m=re.search(r'flush-compress ([0-9.]+)', l)
        if m and float(m.group(1))>15: print(l[:110])
PY
done
