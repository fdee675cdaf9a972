import sys, ctypes as C, torch, numpy as np
sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc
import bench
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = fc.Context(0, stream=stream.cuda_stream)
dev = torch.device('cuda', 0)
for rows in (1000, 100000, 1000000):
    t = bench.make_table(torch, fc, ctx, rows, 768, 2, dev)
    torch.cuda.synchronize()
    n = (t.double()**2).sum(1).sqrt()
    err = (n - 1).abs()
    print(rows, 'max err', err.max().item(), 'argmax', err.argmax().item(), 'nonfinite', (~torch.isfinite(t)).sum().item(), flush=True)
    bad = (err > 1e-6).nonzero().flatten()[:5].tolist()
    print(' bad rows', bad, [n[b].item() for b in bad])
