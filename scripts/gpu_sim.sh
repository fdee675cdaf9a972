timeout -s KILL 600 python -m pytest tests/test_simgen.py tests/test_capi.py -q -x 2>&1 | tail -5
python - <<'PY'
import sys, time; sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc, torch, numpy as np
sets = [[i] for i in range(1_000_000)]
t0 = time.perf_counter(); x = fc.synth_embeddings(sets, 768, 2); torch.cuda.synchronize(); t1 = time.perf_counter()
x = fc.synth_embeddings(sets, 768, 2); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"synth 1M x 768 embeddings: {t2 - t1:.3f} s (first {t1 - t0:.3f} s)")
t0 = time.perf_counter(); lat, om, bm = fc.synth_latents(list(range(256)), 64, (40, 64, 4)); torch.cuda.synchronize()
print(f"synth 256 x 5 x 64 x 40x64x4 latents: {time.perf_counter() - t0:.3f} s")
PY
