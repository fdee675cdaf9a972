import sys, time, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc
import bench
rows, kp, nb = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = fc.Context(0, stream=stream.cuda_stream)
dev = torch.device('cuda', 0)
full = bench.make_table(torch, fc, ctx, rows, 768, 2, dev)
ix = fc.SimilarityIndex(ctx=ctx)
ix.insert_batch(np.arange(rows, dtype=np.uint64), full, full, full)
ix.set_lookup(2, kp)
q = bench.make_queries(torch, fc, ctx, full, nb, 1000, dev)
t0 = time.time()
ids, sc, cnt = ix.query_topk(fc.EmbeddingKind.Whole, q, 8)
torch.cuda.synchronize()
st = ix.stats()
print(f"rows={rows} kp={kp} nq={nb}: {time.time()-t0:.2f}s certified {st.certified} fallback {st.fallback} maxerr {st.max_abs_err:.2e}", flush=True)
