import sys, time, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc
import bench
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
kp = int(sys.argv[2]) if len(sys.argv) > 2 else 32
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 768
nb = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = fc.Context(0, stream=stream.cuda_stream)
dev = torch.device('cuda', 0)
full = bench.make_table(torch, fc, ctx, rows, dim, 2, dev)
ix = fc.SimilarityIndex(ctx=ctx)
ids = np.arange(rows, dtype=np.uint64)
ix.insert_batch(ids, full, full, full)
ix.set_lookup(0, kp)
qs = [bench.make_queries(torch, fc, ctx, full, nb, 1000 + s, dev) for s in range(6)]
out = (torch.empty((nb, 8), dtype=torch.int64, device=dev), torch.empty((nb, 8), dtype=torch.float64, device=dev), torch.empty(nb, dtype=torch.int32, device=dev))
for s in range(2): ix.query_topk(fc.EmbeddingKind.Whole, qs[s], 8, out=out)
torch.cuda.synchronize()
fc.lib.lc_ctx_profile(ctx.h, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for s in range(6): ix.query_topk(fc.EmbeddingKind.Whole, qs[s], 8, out=out)
e1.record(stream); torch.cuda.synchronize()
n_, tot = C.c_uint64(), C.c_double()
fc.lib.lc_ctx_kernel_time(ctx.h, b"shortlist", C.byref(n_), C.byref(tot), 1)
sl = tot.value / n_.value
tf = 2 * nb * rows * dim / (sl / 1e3) / 1e12
st = ix.stats()
parts = []
for name in (b"shortlist_pilot", b"shortlist_merge", b"rescore", b"shortlist_tier2", b"rescore_tier2", b"scan"):
    fc.lib.lc_ctx_kernel_time(ctx.h, name, C.byref(n_), C.byref(tot), 1)
    parts.append(f"{name.decode()} {tot.value / 6:.3f}")
print(f"rows={rows} dim={dim} kp={kp} nq={nb}: step {e0.elapsed_time(e1)/6:.2f} ms, shortlist {sl:.3f} ms = {tf:.0f} T(FL)OP/s, "
      f"fallback {st.fallback} i8 batches {st.i8_batches} cands/query {st.i8_candidates / max(1, 8 * nb):.1f} bf16/query {st.i8_prescored / max(1, 8 * nb):.1f} exact/query {st.i8_rescored / max(1, 8 * nb):.1f} | per step ms: " + ", ".join(parts), flush=True)
