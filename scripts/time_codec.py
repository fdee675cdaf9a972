"""Codec timing breakdown on config[2] (diagnostic): compress kernels + host,
decompress / decompress_stitch kernel GB/s."""
import ctypes as C, sys, time
import torch
sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
F = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dims = tuple(int(x) for x in sys.argv[3].split('x')) if len(sys.argv) > 3 else (40, 64, 4)  # e.g. 72x128x4 (config[4])
E = dims[0] * dims[1] * dims[2]
dev = torch.device('cuda', 0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = fc.Context(0, stream=stream.cuda_stream)
lat, om, bm = bench.make_latents(torch, n, F, dims, 3, dev)
torch.cuda.synchronize()
steps = [5, 10, 15, 20, 25]; prompts = list(range(1, n + 1))
ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx); del ents
names = ("gram", "select", "inter", "pack", "decompress", "decompress_stitch")
def kt(reset=1):
    r = {}
    for nm in names:
        c_, t_ = C.c_uint64(), C.c_double()
        fc.lib.lc_ctx_kernel_time(ctx.h, nm.encode(), C.byref(c_), C.byref(t_), reset)
        if c_.value: r[nm] = round(t_.value, 3)
    return r
fc.lib.lc_ctx_profile(ctx.h, 1); kt()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    raw = n * 5 * F * E * 4
    print(f"compress {dt*1e3:.2f} ms wall = {(raw + int(sizes.sum()))/dt/1e9:.0f} GB/s  kernels {kt()}", flush=True)
    if rep < 2: del ents
out = torch.empty((n, F, E), dtype=torch.float32, device=dev)
for s in steps: fc.decompress_batch(ents, [s] * n, out=out)
kt()
for s in steps: fc.decompress_batch(ents, [s] * n, out=out)
k = kt()
infos = [e.info() for e in ents]
rb = sum(4 * E * (1 + i.n_extra[si]) + 2 * F + 4 * i.n_diff for i in infos for si in range(i.n_steps)) + \
     sum(4 * E * i.n_diff * i.n_steps for i in infos)
tot = n * 5 * F * E * 4 + rb
print(f"decompress: {k.get('decompress')} ms for 5 launches = {tot / (k['decompress'] / 1e3) / 1e9:.0f} GB/s (alg bytes {tot/1e9:.2f} GB)")
half = n // 2
out2 = torch.empty((half, F, E), dtype=torch.float32, device=dev)
fc.decompress_stitch(ents[:half], ents[half:2 * half], [15] * half, out=out2); kt()
fc.decompress_stitch(ents[:half], ents[half:2 * half], [15] * half, out=out2); k = kt()
sb = half * F * E * 4 * 2 + 2 * half * F * (dims[0] * dims[1] // 8)
print(f"decompress_stitch: {k.get('decompress_stitch')} ms = {sb / (k['decompress_stitch'] / 1e3) / 1e9:.0f} GB/s")
