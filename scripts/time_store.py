"""Store timing breakdown (diagnostic): evict_one per-call cost, scoring launches."""
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2501_04012_b200 as fc
n_p = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
ctx = fc.Context(0)
steps = [5, 10, 15, 20, 25]
rng = np.random.default_rng(7)
lat = rng.standard_normal((n_p, 5, 1, 64)).astype(np.float32)
om = np.zeros((n_p, 1, 8), np.uint8)
t0 = time.perf_counter()
ents, sizes = fc.compress_batch(lat, steps, om, om, (8, 8, 1), list(range(1, n_p + 1)), ctx=ctx)
print(f"compress {n_p}: {time.perf_counter()-t0:.2f} s")
st = fc.CacheStore(int(sizes.sum()) * 2, fc.Policy.Lrbu, ctx=ctx)
t0 = time.perf_counter()
for i, e in enumerate(ents):
    st.insert_steps(i + 1, e, steps, i + 1)
print(f"insert {n_p}: {time.perf_counter()-t0:.2f} s")
del ents
now = n_p + 1
if len(sys.argv) > 2 and sys.argv[2] == "gets":  # bench.py's access pattern: vary f / last_access
    for pid in rng.integers(1, n_p + 1, n_p // 2):
        st.get_step(int(pid), 25, now, want_latent=False)
        now += 1
fc.lib.lc_ctx_profile(ctx.h, 1)
for mode in ("py", "raw"):
    e = fc._capi.StepEntry()
    ts = []
    for k in range(1000):
        t0 = time.perf_counter()
        if mode == "py":
            st.evict_one(now)
        else:
            fc._check(fc.lib.lc_store_evict_one(st.h, now, C.byref(e)))
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e6
    c_, t_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy", C.byref(c_), C.byref(t_), 1)
    cc_, tc_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy_call", C.byref(cc_), C.byref(tc_), 1)
    print(f"  scoring call span (launch..readback): {tc_.value / max(1, cc_.value) * 1e3:.1f} us x {cc_.value}")
    print(f"{mode}: median {np.median(ts):.1f} us, mean {ts.mean():.1f} us, max {ts.max():.0f} us; "
          f"scorings {c_.value} x {t_.value / max(1, c_.value):.3f} ms")
