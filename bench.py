#!/usr/bin/env python
"""bench.py — FlexCache B200 hot-path benchmark (driver contract).

Headline (BASELINE.json metric, config[1]): prompt-similarity lookups/s
against a 1M-entry cache, 768-d embeddings, 4096-query batches, top-8,
entries sharded by id mod N over N GPUs (strong scaling; one NCCL all-gather
of the per-shard exact top-8 + merge per batch). One step = one 4096-query
batch. Lookups are EXACT (bit-identical ids/scores to the reference's
sequential fp64 scan): bf16 tcgen05 shortlist + fp64 rescore + certified
margin (+ exact fallback).

Also reported (same JSON line, "codec"): latent codec compress / decompress
GB/s on config[2] (256 prompts x 5 steps x 64 frames x 40x64x4) as a fraction
of the measured HBM roofline.

  python bench.py [--gpus N --steps K --warmup W]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference      # reference CPU implementation arm
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# load every kernel at context creation: a rarely-taken path (exact fallback
# scan) must not pay lazy module loading inside the timed region
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback"
    return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--kprime", type=int, default=32)
    ap.add_argument("--codec-prompts", type=int, default=256)
    ap.add_argument("--codec-frames", type=int, default=64)
    ap.add_argument("--no-codec", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the config[4] large-latent section")
    ap.add_argument("--large-prompts", type=int, default=32)
    ap.add_argument("--no-scoring", action="store_true")
    ap.add_argument("--score-prompts", type=int, default=100_000)
    ap.add_argument("--score-evictions", type=int, default=2000)
    ap.add_argument("--no-engine", action="store_true")
    ap.add_argument("--engine-cached", type=int, default=10_000)
    ap.add_argument("--engine-requests", type=int, default=1000)
    ap.add_argument("--mixed-requests", type=int, default=16384)
    ap.add_argument("--mixed-capacity-gb", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=0, help="reference sample size (0 = auto)")
    ap.add_argument("--seed", type=int, default=2)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (nvidia-smi's 100 ms loop misses a ~0.1 s region)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                        self.rows.append((sm, rs, util))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[1] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "sampler": "nvml, 2 ms"}


# ---------------------------------------------------------------------------
# synthetic inputs on the device
# ---------------------------------------------------------------------------
def make_table(torch, fc, ctx, rows, dim, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    raw = torch.randn(rows, dim, generator=g, device=dev, dtype=torch.float32)
    out = torch.empty_like(raw)
    fc._check(fc.lib.lc_embedding_normalize(ctx.h, C.c_void_p(raw.data_ptr()), rows, dim, C.c_void_p(out.data_ptr())))
    del raw
    # 5% exact duplicates of earlier rows: id tie-breaks are exercised
    nd = rows // 20
    src = torch.randint(0, rows // 2, (nd,), generator=g, device=dev)
    dst = rows // 2 + torch.randperm(rows - rows // 2, generator=g, device=dev)[:nd]  # unique targets
    out[dst] = out[src]
    return out


def make_queries(torch, fc, ctx, table, n, seed, dev):
    """50% fresh unit Gaussians (misses), 50% stored rows moved by sigma*u,
    sigma ~ U[0, 1.25] (hits over all five step bins)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    dim = table.shape[1]
    q = torch.randn(n, dim, generator=g, device=dev)
    h = n // 2
    src = torch.randint(0, table.shape[0], (h,), generator=g, device=dev)
    u = torch.randn(h, dim, generator=g, device=dev)
    u = u / u.norm(dim=1, keepdim=True)
    sig = torch.rand(h, 1, generator=g, device=dev) * 1.25
    q[:h] = table[src] + sig * u
    q = q[torch.randperm(n, generator=g, device=dev)].contiguous()
    out = torch.empty_like(q)
    fc._check(fc.lib.lc_embedding_normalize(ctx.h, C.c_void_p(q.data_ptr()), n, dim, C.c_void_p(out.data_ptr())))
    return out


def make_latents(torch, n, F, dims, seed, dev):
    """Device restatement of synth.latents (config[2]): per step a first
    frame, shared differential fields scaled by the alpha schedule with 1%
    relative noise, nested redundant frames (near-copies, 2% jitter)."""
    H, W, Cc = dims
    E = H * W * Cc
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    red = (0.9, 0.8, 0.6, 0.4, 0.25)
    alph = (1.0, 0.9, 0.8, 0.7, 0.6)
    base = torch.randn(n, E, generator=g, device=dev)
    D = torch.randn(n, F, E, generator=g, device=dev)
    order = torch.argsort(torch.rand(n, F - 1, generator=g, device=dev), dim=1) + 1  # nested redundancy order
    rank = torch.empty_like(order)
    rank.scatter_(1, order - 1, torch.arange(F - 1, device=dev).expand(n, F - 1).contiguous())
    out = torch.empty(n, 5, F, E, device=dev)
    for i in range(5):
        first = base * (1 - 0.05 * i) + 0.05 * torch.randn(n, E, generator=g, device=dev)
        n_red = int(round(red[i] * (F - 1)))
        out[:, i, 0] = first
        for j in range(1, F):
            is_red = (rank[:, j - 1] < n_red).view(n, 1)
            key = first + alph[i] * D[:, j] * (1 + 0.01 * torch.randn(n, E, generator=g, device=dev))
            prev = out[:, i, j - 1]
            dup = prev + (0.02 / E ** 0.5) * prev.norm(dim=1, keepdim=True) * torch.randn(n, E, generator=g, device=dev)
            out[:, i, j] = torch.where(is_red, dup, key)
    # rectangular object masks drifting one pixel per frame, background = complement
    hh = torch.randint(1, H, (n, 2), generator=g, device=dev).sort(dim=1).values
    ww = torch.randint(1, W // 2, (n, 2), generator=g, device=dev).sort(dim=1).values
    ys = torch.arange(H, device=dev).view(1, 1, H, 1)
    xs = torch.arange(W, device=dev).view(1, 1, 1, W)
    fr = torch.arange(F, device=dev).view(1, F, 1, 1)
    obj = ((ys >= hh[:, 0].view(n, 1, 1, 1)) & (ys < hh[:, 1].view(n, 1, 1, 1) + 1) &
           (xs >= ww[:, 0].view(n, 1, 1, 1) + fr % 8) & (xs < ww[:, 1].view(n, 1, 1, 1) + 1 + fr % 8))
    bits = obj.view(n, F, H * W // 8, 8).to(torch.uint8)
    wts = (2 ** torch.arange(8, device=dev, dtype=torch.uint8)).view(1, 1, 1, 8)
    om = (bits * wts).sum(dim=3, dtype=torch.uint8).contiguous()
    bm = ((1 - bits) * wts).sum(dim=3, dtype=torch.uint8).contiguous()
    return out.contiguous(), om, bm


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------
def cpu_reference_lookup(table_np, queries_np, nthreads, n_q):
    """query_top1 of the UNMODIFIED reference (oracle/_ref) on host cores —
    or the plain-C restatement when the reference library is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Checker, available
    kind = "reference" if available("ref") else "port"
    chk = Checker("ref" if kind == "reference" else "orc")
    dim = table_np.shape[1]
    ix = chk.index(dim)
    t0 = time.perf_counter()
    lib = chk.lib
    fn = getattr(lib, chk.pfx + "index_insert")
    base = table_np.ctypes.data
    rowb = dim * 4
    for i in range(table_np.shape[0]):
        p = C.c_void_p(base + i * rowb)
        rc = fn(ix.h, i, p, p, p, dim)
        if rc:
            raise RuntimeError(chk._f("last_error")())
    build_s = time.perf_counter() - t0
    q = np.ascontiguousarray(queries_np[:n_q])
    t0 = time.perf_counter()
    rid, rsc, _ = ix.query_top1(0, q, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return kind, n_q / dt, build_s, dt, (rid, rsc)


def _safe(fn):
    try:
        return fn()
    except Exception as ex:  # reported, never the target
        return {"value": None, "kind": "unavailable", "sample": str(ex)[:200]}


def cpu_reference_codec(lat_np, om_np, bm_np, nthreads):
    """The reference's intra_compress x 5 + inter_compress (oracle/_ref) on
    host cores over a bounded sample of the config[2] prompts."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Checker, available
    kind = "reference" if available("ref") else "port"
    chk = Checker("ref" if kind == "reference" else "orc")
    n = lat_np.shape[0]
    t0 = time.perf_counter()
    hashes = None
    if kind == "reference":  # sizes + a weighted byte sum of each entry's wire bytes (checked below)
        sizes, hashes = chk.compress_batch_hash(lat_np, [5, 10, 15, 20, 25], om_np, bm_np, (40, 64, 4),
                                                list(range(1, n + 1)), nthreads=nthreads)
    else:
        sizes = chk.compress_batch_sizes(lat_np, [5, 10, 15, 20, 25], om_np, bm_np, (40, 64, 4),
                                         list(range(1, n + 1)), nthreads=nthreads)
    dt = time.perf_counter() - t0
    byt = lat_np.nbytes + om_np.nbytes + bm_np.nbytes + int(sizes.sum())
    return {"value": byt / dt / 1e9, "unit": "GB/s (compress)", "cores": nthreads, "kind": kind,
            "sample": f"{n} config[2] prompts (5 x 64 x 40x64x4), {dt:.1f}s"}, sizes, hashes


def wire_sum(b):
    """The weighted byte sum the reference's compress_batch_hash reports (oracle/ref_shim.cpp)."""
    b = np.frombuffer(b, np.uint8).astype(np.uint64)
    w = (np.arange(b.size, dtype=np.uint64) * np.uint64(0x9E3779B1) + np.uint64(1)) & np.uint64(0xFFFFFFFF)
    return int((b * w).sum(dtype=np.uint64))


def cpu_reference_evict(n_prompts=100_000, n_ev=16):
    """The reference's evict_one (single writer, store.cpp:113-157) at
    5 x n_prompts live steps (bench_scoring's state, without get_steps)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Checker, available
    kind = "reference" if available("ref") else "port"
    chk = Checker("ref" if kind == "reference" else "orc")
    rng = np.random.default_rng(7)
    lat = rng.standard_normal((1, 5, 1, 64)).astype(np.float32)
    om = np.zeros((1, 8), np.uint8)
    st = chk.store(1 << 62, 3)
    steps = [5, 10, 15, 20, 25]
    ent = chk.compress(lat[0], steps, om, om, (8, 8, 1), 1)
    # the same bytes for every prompt id: patch the prompt field (first 8 bytes, LE)
    t0 = time.perf_counter()
    for i in range(n_prompts):
        b = (i + 1).to_bytes(8, "little") + ent[8:]
        st.insert(i + 1, b, steps, i + 1)
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(n_ev):
        st.evict_one(n_prompts + 1)
    dt = time.perf_counter() - t0
    return {"value": n_ev / dt, "unit": "evictions/s", "cores": 1, "kind": kind,
            "ms_per_evict_one": dt / n_ev * 1e3,
            "sample": f"{n_ev} evict_one at {5 * n_prompts} live steps (LRBU); store build {build_s:.1f}s excluded"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rng = np.random.default_rng(args.seed)
    sys.path.insert(0, os.path.join(ROOT, "paper_2501_04012_b200"))
    import importlib.util
    spec = importlib.util.spec_from_file_location("synth", os.path.join(ROOT, "paper_2501_04012_b200", "synth.py"))
    synth = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(synth)
    rows = args.rows
    tab = rng.standard_normal((rows, args.dim), dtype=np.float32)
    tab = synth.normalize_rows(tab)
    qs, _ = synth.perturbed_queries(tab, 4096, args.seed + 1)
    nthreads = os.cpu_count() or 1
    per_step = args.cpu_queries or max(nthreads, 8)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Checker, available
    kind = "reference" if available("ref") else "port"
    chk = Checker("ref" if kind == "reference" else "orc")
    ix = chk.index(args.dim)
    fn = getattr(chk.lib, chk.pfx + "index_insert")
    base = tab.ctypes.data
    for i in range(rows):
        p = C.c_void_p(base + i * args.dim * 4)
        if fn(ix.h, i, p, p, p, args.dim):
            raise RuntimeError("reference insert failed")
    times = []
    for s in range(args.warmup + args.steps):
        q = qs[(s * per_step) % (4096 - per_step):][:per_step]
        t0 = time.perf_counter()
        ix.query_top1(0, q, nthreads=nthreads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = per_step * len(times) / total
    line = {"impl": "reference", "metric": "cache lookups/s @1M entries", "value": value, "unit": "lookups/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * total / len(times), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config[1] lookup: 1M cached 768-d embeddings, top-1 (reference query_top1)",
                       "rows": rows, "dim": args.dim, "queries_per_step": per_step},
            "cpu_baseline": {"value": value, "unit": "lookups/s", "cores": nthreads, "kind": kind,
                             "sample": f"{per_step} queries per step x {args.steps} steps, query_top1 over "
                                       f"{rows} rows, {nthreads} concurrent readers"},
            "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; FC_DIST_BACKEND=gloo lets several ranks share one GPU (smoke runs)
    backend = os.environ.get("FC_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2501_04012_b200 as fc
    stream = torch.cuda.Stream(device=dev)  # library + collectives + events share this stream
    torch.cuda.set_stream(stream)
    ctx = fc.Context(local, stream=stream.cuda_stream)
    peaks = load_peaks()

    # ---- index shard: ids = r (mod world) ----
    full = make_table(torch, fc, ctx, args.rows, args.dim, args.seed, dev)
    ids_all = torch.arange(args.rows, device=dev, dtype=torch.int64)
    mine = (ids_all % world) == rank
    shard_ids = ids_all[mine].contiguous()
    n_local = int(shard_ids.numel())
    ix = fc.SimilarityIndex(ctx=ctx)
    tabs = []
    for t in range(3):
        tt = full[mine].contiguous() if t == 0 else make_table(torch, fc, ctx, args.rows, args.dim,
                                                               args.seed + 100 * t, dev)[mine].contiguous()
        tabs.append(tt)
    ix.insert_batch(shard_ids.cpu().numpy().astype(np.uint64), tabs[0], tabs[1], tabs[2])
    del tabs
    ix.set_lookup(0, args.kprime)
    nb = args.warmup + args.steps
    qs = [make_queries(torch, fc, ctx, full, args.batch, 1000 + s, dev) for s in range(nb)]
    k = args.k
    B = args.batch
    o_ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    o_sc = torch.empty((B, k), dtype=torch.float64, device=dev)
    o_cnt = torch.empty((B,), dtype=torch.int32, device=dev)
    last = {}
    comm = None
    if world > 1:
        # the communicator lives in the library context (lc_ctx_comm_init:
        # NCCL over NVLink; host transport through the gloo group for
        # FC_DIST_BACKEND=gloo smoke runs); each batch = local exact top-k,
        # one grouped all-gather, k_topk_merge (lc_sharded_query_topk)
        from paper_2501_04012_b200 import sharded
        sharded.attach_comm(ctx, transport="nccl" if backend == "nccl" else "host")
        shard = sharded.CommShardedIndex(ix, args.dim)
        nr, rk, be, _ = sharded.comm_info(ctx)
        comm = {"backend": {1: "nccl", 2: "host"}.get(be, "none"), "nranks": nr, "rank": rk,
                "api": "lc_sharded_query_topk"}

    def step(q):
        if world > 1:
            last["res"] = shard.query_topk(fc.EmbeddingKind.Whole, q, k, out=(o_ids, o_sc, o_cnt))
        else:
            ix.query_topk(fc.EmbeddingKind.Whole, q, k, out=(o_ids, o_sc, o_cnt))
            last["res"] = (o_ids, o_sc, o_cnt)

    for s in range(args.warmup):
        step(qs[s])
    ix.stats(reset=True)
    fc.lib.lc_ctx_profile(ctx.h, 1)
    for name in ("shortlist", "shortlist_pilot", "rescore", "scan", "shortlist_tier2", "rescore_tier2", "shortlist_merge"):
        fc.lib.lc_ctx_kernel_time(ctx.h, name.encode(), None, None, 1)
    launches0 = ctx.launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        ev0.record(stream)
        evs[0].record(stream)
        for i, s in enumerate(range(args.warmup, nb)):
            step(qs[s])
            evs[i + 1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    if world > 1:
        dist.barrier()
    fc.lib.lc_ctx_profile(ctx.h, 0)
    launches = ctx.launches - launches0
    ms = ev0.elapsed_time(ev1)
    red_dev = dev if backend == "nccl" else "cpu"
    t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps * B / (ms / 1000.0)
    st = ix.stats()
    kt = {}
    for name in ("shortlist", "shortlist_pilot", "rescore", "scan", "shortlist_tier2", "rescore_tier2", "shortlist_merge"):
        n_, tot = C.c_uint64(), C.c_double()
        fc.lib.lc_ctx_kernel_time(ctx.h, name.encode(), C.byref(n_), C.byref(tot), 1)
        kt[name] = (n_.value, tot.value)

    # roofline of the dominant kernel (tcgen05 shortlist GEMM: the s8 tier-1
    # pass when the int8 tier ran, else the bf16 pass)
    n_sl, t_sl = kt["shortlist"]
    flops_per_launch = 2.0 * B * n_local * args.dim
    roof = None
    i8_tier = st.i8_batches > 0
    if n_sl:
        avg = t_sl / n_sl
        achieved = flops_per_launch / (avg / 1000.0) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "shortlist_i8_traffic.json" if i8_tier else "shortlist_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        if i8_tier:
            # s8 dense tensor rate = 2x bf16 on sm_100 (nominal 4.5 vs 2.25 P; the
            # issue-rate microbenchmark measured 2.08x, profiles/r02p_mma_i8_rates.log):
            # the denominator is twice the measured cuBLAS bf16 burst figure
            peak = 2.0 * peaks["bf16_tflops"]
            roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": "TOPS (s8)",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "kernel": "k_shortlist_pair<int8> (tcgen05 kind::i8, cta_group::2)",
                    "avg_launch_ms": round(avg, 4),
                    "peak_source": peaks["source"] + " 2 x bf16_tflops (burst); s8 = 2x bf16 dense",
                    "frac_of_sustained": round(achieved / (2.0 * peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])), 4),
                    "frac_of_mma_microbench": round(achieved / 4138.5, 4),
                    "kernel_share_of_step": round(t_sl / ms, 4)}
        else:
            peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
            roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": "k_shortlist (tcgen05)",
                    "avg_launch_ms": round(avg, 4), "peak_source": peaks["source"] + " bf16_tflops_sustained",
                    "frac_of_burst": round(achieved / peaks["bf16_tflops"], 4),
                    "kernel_share_of_step": round(t_sl / ms, 4)}

    # ---- e2e: same lookups through the public API with HOST buffers ----
    e2e = None
    if world == 1:
        hq = [torch.empty((B, args.dim), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        for i in range(2):
            hq[i].copy_(qs[i])
        hid = np.zeros((B, k), np.uint64)
        hsc = np.zeros((B, k), np.float64)
        hcnt = np.zeros(B, np.int32)
        qptrs = [C.c_void_p(h.data_ptr()) for h in hq]
        fn = fc.lib.lc_index_query_topk
        for i in range(2):
            fc._check(fn(ix.h, 0, qptrs[i], B, k, hid.ctypes.data_as(C.c_void_p), hsc.ctypes.data_as(C.c_void_p),
                         hcnt.ctypes.data_as(C.c_void_p)))
        t0 = time.perf_counter()
        for s in range(args.steps):
            fc._check(fn(ix.h, 0, qptrs[s % 2], B, k, hid.ctypes.data_as(C.c_void_p), hsc.ctypes.data_as(C.c_void_p),
                         hcnt.ctypes.data_as(C.c_void_p)))
        e2e_s = time.perf_counter() - t0
        e2e = {"value": args.steps * B / e2e_s, "unit": "lookups/s", "h2d_bytes_per_step": B * args.dim * 4,
               "d2h_bytes_per_step": B * k * 16 + B * 4, "api": "lc_index_query_topk (host pointers)"}
    else:
        hq = torch.empty((B, args.dim), dtype=torch.float32, pin_memory=True)
        hq.copy_(qs[0])
        hres = torch.empty((B, k), dtype=torch.int64, pin_memory=True)
        dq = torch.empty((B, args.dim), dtype=torch.float32, device=dev)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                dq.copy_(hq, non_blocking=True)
            step(dq)
            with torch.cuda.stream(stream):
                hres.copy_(last["res"][0], non_blocking=True)
            stream.synchronize()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": args.steps * B / float(tt.item()), "unit": "lookups/s",
               "h2d_bytes_per_step": B * args.dim * 4, "d2h_bytes_per_step": B * k * 8,
               "api": f"lc_sharded_query_topk: local exact top-k + one {backend} all-gather + k_topk_merge, "
                      "pinned host queries"}

    # ---- codec (config[2]) ----
    codec = None
    if not args.no_codec and rank == 0:
        codec = bench_codec(torch, fc, ctx, args, dev, peaks)

    large = None
    if not args.no_codec and not args.no_large and rank == 0:
        try:
            large = bench_codec_large(torch, fc, ctx, args, dev, peaks)
        except Exception as ex:  # reported, never fatal to the headline line
            large = {"error": str(ex)[:200]}

    scoring = None
    if not args.no_scoring and rank == 0:
        try:
            scoring = bench_scoring(torch, fc, ctx, args, peaks)
        except Exception as ex:  # reported, never fatal to the headline line
            scoring = {"error": str(ex)[:200]}

    engine = None
    if not args.no_engine and rank == 0:
        try:
            engine = bench_engine(torch, fc, ctx, args, dev)
            engine["mixed"] = bench_engine_mixed(torch, fc, ctx, args, dev)
        except Exception as ex:  # reported, never fatal to the headline line
            engine = {"error": str(ex)[:200]}

    # ---- CPU baseline: reference query_top1 on this box's host cores ----
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            nthreads = os.cpu_count() or 1
            n_q = args.cpu_queries or max(2 * nthreads, 16)
            tab_np = full.cpu().numpy()
            q_np = qs[0][:n_q].cpu().numpy()
            del full
            kind, v, build_s, dt, (rid, rsc) = cpu_reference_lookup(tab_np, q_np, nthreads, n_q)
            cpu = {"value": v, "unit": "lookups/s", "cores": nthreads, "kind": kind,
                   "sample": f"{n_q} queries x query_top1 over {args.rows} rows (whole table), {nthreads} "
                             f"concurrent readers; index build {build_s:.1f}s excluded; {dt:.1f}s timed"}
            # the timed path's answers for the same queries (batch qs[0], re-run
            # untimed through the int8 tier) against the reference's query_top1
            step(qs[0])
            torch.cuda.synchronize()
            gid = o_ids[:n_q, 0].cpu().numpy().view(np.uint64)
            gsc = o_sc[:n_q, 0].cpu().numpy()
            same = (gid == rid) & (gsc.view(np.uint64) == rsc.view(np.uint64))
            cpu["parity"] = {"queries": int(n_q), "top1_identical": int(same.sum()),
                             "vs": f"{kind} query_top1 (ids and fp64 scores, bitwise)"}
        except Exception as ex:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "lookups/s", "cores": 0, "kind": "unavailable", "sample": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": "cache lookups/s @1M entries", "value": value, "unit": "lookups/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "ms_per_step_median": statistics.median(step_ms), "ms_per_step_max": max(step_ms),
            "ms_per_step_all": [round(x, 3) for x in step_ms], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "s8 tensor-core candidates, f64 exact scores" if i8_tier else "bf16 tensor-core candidates, f64 exact scores",
            "data": "synthetic",
            "config": {"workload": f"config[1] lookup: {args.rows:,} cached {args.dim}-d embeddings, {B}-query batches, "
                                   f"top-{k}",
                       "rows": args.rows, "dim": args.dim, "global_batch": B, "k": k, "kprime": args.kprime,
                       "sharding": f"id mod {world}", "parallelism": f"entry-sharded x{world}",
                       "l2": "inputs larger than L2 (1.5 GB bf16 table streamed per step)",
                       "exactness": "bit-exact top-8 vs the fp64 reference scan: certified int8 shortlist "
                                    "(bf16 tier and exact scan behind it)" if i8_tier else
                                    "bit-exact top-8 vs fp64 reference scan (certified bf16 shortlist)"},
            "lookup_stats": {"certified": st.certified, "fallback": st.fallback, "max_abs_err": st.max_abs_err,
                             "tier2_certified": st.tier2_certified, "exact_scans": st.exact_scans,
                             "i8_batches": st.i8_batches,
                             "i8_candidates_per_query": st.i8_candidates / max(1, st.queries),
                             "i8_prescored_per_query": st.i8_prescored / max(1, st.queries),
                             "i8_exact_per_query": st.i8_rescored / max(1, st.queries)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(), "kernel_ms": {k_: round(v_[1], 3) for k_, v_ in kt.items()},
            "codec": codec, "codec_large": large, "scoring": scoring, "engine": engine, "comm": comm,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_codec(torch, fc, ctx, args, dev, peaks):
    n, F = args.codec_prompts, args.codec_frames
    dims = (40, 64, 4)
    E = 40 * 64 * 4
    lat, om, bm = make_latents(torch, n, F, dims, 3, dev)
    torch.cuda.synchronize()
    steps = [5, 10, 15, 20, 25]
    prompts = list(range(1, n + 1))
    ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx)  # warm-up
    del ents
    fc.lib.lc_ctx_profile(ctx.h, 1)
    for name in ("gram", "inter", "pack", "decompress", "decompress_stitch"):
        fc.lib.lc_ctx_kernel_time(ctx.h, name.encode(), None, None, 1)
    reps = 5
    rep_s = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx)
        rep_s.append(time.perf_counter() - t0)
        if _ < reps - 1:
            del ents
    comp_s = statistics.median(rep_s)  # one call per rep; the median resists a one-off host stall
    raw = n * 5 * F * E * 4
    mask_b = 2 * n * F * (40 * 64 // 8)
    comp_bytes = raw + mask_b + int(sizes.sum())
    out = torch.empty((n, F, E), dtype=torch.float32, device=dev)
    for s in steps:  # warm-up
        fc.decompress_batch(ents, [s] * n, out=out)
    c_, t_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"decompress", None, None, 1)  # drop the warm-up launches
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec_reps = 2
    for _ in range(dec_reps):
        for s in steps:
            fc.decompress_batch(ents, [s] * n, out=out)
    torch.cuda.synchronize()  # the decompress calls are stream-ordered
    dec_s = (time.perf_counter() - t0) / dec_reps
    # kernel time of exactly these dec_reps x 5 launches (before the fidelity pass adds more)
    dk_c, dk_tt = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"decompress", C.byref(dk_c), C.byref(dk_tt), 1)
    # fidelity of the served latents vs the raw ones (outside the timed region):
    # the codec is lossy by design (non-key frames are served as their key
    # frame, non-base steps as first + alpha * diff), bounded per frame by the
    # key-frame threshold (select_keyframes, codec.cpp:138-165)
    fid = {"max_abs": 0.0, "sq_err": 0.0, "sq_ref": 0.0, "cos_min": 1.0, "cos_sum": 0.0, "frames": 0,
           "frames_ge_thr": 0}
    for si, s_ in enumerate(steps):
        fc.decompress_batch(ents, [s_] * n, out=out)
        ref_ = lat[:, si]
        d_ = (out - ref_).double()
        fid["max_abs"] = max(fid["max_abs"], float(d_.abs().max()))
        fid["sq_err"] += float((d_ * d_).sum())
        rd = ref_.double()
        od = out.double()
        fid["sq_ref"] += float((rd * rd).sum())
        cos = (od * rd).sum(-1) / (od.norm(dim=-1) * rd.norm(dim=-1))
        fid["cos_min"] = min(fid["cos_min"], float(cos.min()))
        fid["cos_sum"] += float(cos.sum())
        fid["frames"] += cos.numel()
        fid["frames_ge_thr"] += int((cos >= 0.99).sum())
        del d_, rd, od, cos
    fidelity = {"max_abs": fid["max_abs"], "rel_l2": (fid["sq_err"] / fid["sq_ref"]) ** 0.5,
                "frame_cosine_min": fid["cos_min"], "frame_cosine_mean": fid["cos_sum"] / fid["frames"],
                "frames_cosine_ge_0.99": fid["frames_ge_thr"] / fid["frames"],
                "vs": "decompress_step (codec.cpp:263-301) of every step vs the raw input latents, fp64 metrics"}
    # algorithmic bytes: every output frame written once + the step's stored data read once
    infos = [e.info() for e in ents]
    read_b = 0
    for i in infos:
        for si in range(i.n_steps):
            read_b += 4 * E * (1 + i.n_extra[si]) + 2 * F + 4 * i.n_diff
        read_b += 4 * E * i.n_diff * (i.n_steps)  # base diffs re-read per step
    dec_bytes = n * 5 * F * E * 4 + read_b
    ker = {}
    for name in ("gram", "inter", "pack"):
        c_, t_ = C.c_uint64(), C.c_double()
        fc.lib.lc_ctx_kernel_time(ctx.h, name.encode(), C.byref(c_), C.byref(t_), 1)
        ker[name] = (c_.value, t_.value)
    ker["decompress"] = (dk_c.value, dk_tt.value)
    # fused decoupled-hit path: decompress(obj) + decompress(bg) + stitch
    half = n // 2
    out2 = torch.empty((half, F, E), dtype=torch.float32, device=dev)
    fc.decompress_stitch(ents[:half], ents[half:2 * half], [15] * half, out=out2)
    c_, t_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"decompress_stitch", None, None, 1)
    fc.decompress_stitch(ents[:half], ents[half:2 * half], [15] * half, out=out2)
    fc.lib.lc_ctx_kernel_time(ctx.h, b"decompress_stitch", C.byref(c_), C.byref(t_), 1)
    fc.lib.lc_ctx_profile(ctx.h, 0)
    hbm = peaks["hbm_gbs"]
    dk_n, dk_t = ker["decompress"]
    dk_bytes = dec_bytes / 5 if dk_n else 0
    dk_gbs = (dec_bytes * dec_reps) / (dk_t / 1000) / 1e9 if dk_t else None
    stitch_bytes = half * F * E * 4 * 2 + 2 * half * F * (40 * 64 // 8)  # out + selected source reads + masks
    dec_traffic = None  # ncu dram read + write per launch (profiles/, one --set full capture), if present
    tpath = os.path.join(ROOT, "profiles", "decompress_traffic.json")
    if os.path.exists(tpath) and n == 256 and F == 64:
        dec_traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
    cpu = None
    if not args.no_cpu:
        try:
            m = min(n, 32)
            cpu, rsz, rh = cpu_reference_codec(lat[:m].cpu().numpy(), om[:m].cpu().numpy(), bm[:m].cpu().numpy(),
                                               os.cpu_count() or 1)
            # the timed compress's entries for the same prompts against the reference's
            same = [int(sizes[i]) == int(rsz[i]) and (rh is None or wire_sum(ents[i].serialize()) == int(rh[i]))
                    for i in range(m)]
            cpu["parity"] = {"prompts": m, "entries_identical": int(sum(same)),
                             "vs": f"{cpu['kind']} compress (sizes" + (" + wire-byte sums)" if rh is not None else ")")}
        except Exception as ex:  # reported, never the target
            cpu = {"value": None, "kind": "unavailable", "sample": str(ex)[:200]}
    res = {
        "cpu_baseline": cpu,
        "workload": f"config[2]: {n} prompts x 5 steps x {F} frames x 40x64x4 fp32, rect masks, thr 0.99",
        "raw_bytes": raw, "compressed_bytes": int(sizes.sum()), "ratio": raw / float(sizes.sum()),
        "compress_GBps": comp_bytes / comp_s / 1e9, "compress_frac_hbm": comp_bytes / comp_s / 1e9 / hbm,
        "compress_s": comp_s, "compress_s_reps": [round(x, 5) for x in rep_s],
        "compress_kernel_ms": {k_: round(v_[1] / max(1, reps), 3) for k_, v_ in ker.items() if k_ != "decompress"},
        "compress_timing": "median of 5 calls, wall clock, inputs device-resident",
        "decompress_GBps_e2e": dec_bytes / dec_s / 1e9, "decompress_frac_hbm_e2e": dec_bytes / dec_s / 1e9 / hbm,
        "roofline": {"bound": "hbm", "achieved": round(dk_gbs, 1) if dk_gbs else None, "peak": hbm, "unit": "GB/s",
                     "frac": round(dk_gbs / hbm, 4) if dk_gbs else None, "traffic": dec_traffic,
                     "kernel": "k_decompress_groups", "bytes_per_launch": int(dk_bytes),
                     "avg_launch_ms": round(dk_t / dk_n, 4) if dk_n else None},
        "decompress_stitch_GBps": (stitch_bytes / (t_.value / 1000) / 1e9) if t_.value else None,
        "fidelity": fidelity,
    }
    return res


def bench_codec_large(torch, fc, ctx, args, dev, peaks):
    """config[4] large-latent stress on one GPU: compress + decompress of
    64-frame 4x72x128 (576x1024 px) latents at batch scale, and the per-step
    cache checkpoint (save_snapshot, store.cpp:232-274, with serialize_entry,
    codec.cpp:358-392) of a store holding them -- written to /dev/shm so the
    number is the serializer's, not a disk's. (The 200k-entry, 8-GPU size of
    config[4] is 25k entries per GPU: scripts/config3_scale.py --dims 72x128x4
    runs that share through the engine with periodic whole-cache checkpoints,
    profiles/r02bf_config4_25k.json.)"""
    import tempfile
    n, F = args.large_prompts, 64
    dims = (72, 128, 4)
    E = 72 * 128 * 4
    steps = [5, 10, 15, 20, 25]
    lat, om, bm = make_latents(torch, n, F, dims, 11, dev)
    torch.cuda.synchronize()
    prompts = list(range(1, n + 1))
    ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx)  # warm-up
    del ents
    reps = 3
    rs = []
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ents, sizes = fc.compress_batch(lat, steps, om, bm, dims, prompts, ctx=ctx)
        rs.append(time.perf_counter() - t0)
        if i < reps - 1:
            del ents
    comp_s = statistics.median(rs)
    raw = n * 5 * F * E * 4
    mask_b = 2 * n * F * (72 * 128 // 8)
    comp_bytes = raw + mask_b + int(sizes.sum())
    out = torch.empty((n, F, E), dtype=torch.float32, device=dev)
    for s_ in steps:
        fc.decompress_batch(ents, [s_] * n, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s_ in steps:
        fc.decompress_batch(ents, [s_] * n, out=out)
    torch.cuda.synchronize()  # the decompress calls are stream-ordered
    dec_s = time.perf_counter() - t0
    infos = [e.info() for e in ents]
    read_b = 0
    for i in infos:
        for si in range(i.n_steps):
            read_b += 4 * E * (1 + i.n_extra[si]) + 2 * F + 4 * i.n_diff
        read_b += 4 * E * i.n_diff * i.n_steps
    dec_bytes = n * 5 * F * E * 4 + read_b
    # checkpoint: store + index holding the n entries, saved after the insert batch
    st = fc.CacheStore(1 << 40, fc.Policy.Lrbu, ctx=ctx)
    for i, e in enumerate(ents):
        st.insert_steps(i + 1, e, steps, i + 1)
    ix = fc.SimilarityIndex(ctx=ctx)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    emb = [make_table(torch, fc, ctx, n, 768, 100 + t, dev) for t in range(3)]
    ix.insert_batch(np.arange(1, n + 1, dtype=np.uint64), *emb)
    shm = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=shm) as td:
        path = os.path.join(td, "ckpt.flxc")
        fc.save_snapshot(st, ix, path)  # warm-up
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fc.save_snapshot(st, ix, path)
            ts.append(time.perf_counter() - t0)
        snap_b = os.path.getsize(path)
        t0 = time.perf_counter()
        st2, ix2 = fc.load_snapshot(path, ctx=ctx)
        load_s = time.perf_counter() - t0
        ok = st2.used() == st.used() and ix2.size() == ix.size()
        del st2, ix2
    save_s = statistics.median(ts)
    hbm = peaks["hbm_gbs"]
    return {"workload": f"config[4] per GPU: {n} prompts x 5 steps x {F} frames x 72x128x4 fp32 "
                        f"({raw / 1e9:.2f} GB raw), rect masks, thr 0.99",
            "compress_GBps": comp_bytes / comp_s / 1e9, "compress_frac_hbm": comp_bytes / comp_s / 1e9 / hbm,
            "compress_s": comp_s, "ratio": raw / float(sizes.sum()),
            "decompress_GBps_e2e": dec_bytes / dec_s / 1e9, "decompress_frac_hbm_e2e": dec_bytes / dec_s / 1e9 / hbm,
            "checkpoint": {"api": "lc_snapshot_save (FLXC v1, byte-identical to the reference's save_snapshot)",
                           "bytes": snap_b, "save_s": save_s, "save_GBps": snap_b / save_s / 1e9,
                           "load_s": load_s, "load_GBps": snap_b / load_s / 1e9, "roundtrip_ok": bool(ok),
                           "target": "/dev/shm" if shm else "tmp"},
            "timing": "wall clock through the public API; compress median of 3 calls, decompress 5 steps x n"}


def bench_engine(torch, fc, ctx, args, dev):
    """config[0] end to end through the engine: a store +
    index pre-populated with N cached prompts (768-d, 16-frame 40x64x4
    latents) drawn from a 50 x 40 object x background template grid, then a
    Zipf(1.0) trace of R requests (fresh embedding noise per request, own
    latents for the cache update) in batches of 64. Reported: requests/s
    (wall, host arrays in), the hit mix and the simulated savings."""
    n_c, n_r, D, F, dims = args.engine_cached, args.engine_requests, 768, 16, (40, 64, 4)
    E = 40 * 64 * 4
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    O = torch.randn(50, D, generator=g, device=dev)
    Bk = torch.randn(40, D, generator=g, device=dev)

    def embs(ti, tk, noise):
        n = ti.numel()
        out = []
        for base in ((O[ti] + Bk[tk]) * 0.7071, O[ti], Bk[tk]):
            raw = (base + noise * torch.randn(n, D, generator=g, device=dev)).contiguous()
            u = torch.empty_like(raw)
            fc._check(fc.lib.lc_embedding_normalize(ctx.h, C.c_void_p(raw.data_ptr()), n, D, C.c_void_p(u.data_ptr())))
            out.append(u)
        return out

    cfg = fc.engine_config(dim=D, F=F, H=40, W=64, C=4, policy=int(fc.Policy.Lrbu))
    eng = fc.Engine(cfg, ctx=ctx)
    # pre-populate N prompts: compress in chunks, insert into the engine's store + index
    tpl = torch.randint(0, 2000, (n_c,), generator=g, device=dev)
    ti, tk = tpl // 40, tpl % 40
    ew, eo, eb = embs(ti, tk, 0.05)
    st, ix = eng.store, eng.index
    t0 = time.perf_counter()
    steps = [5, 10, 15, 20, 25]
    for c0 in range(0, n_c, 512):
        m = min(512, n_c - c0)
        lat, om, bm = make_latents(torch, m, F, dims, 100 + c0, dev)
        ents, _ = fc.compress_batch(lat, steps, om, bm, dims, list(range(c0 + 1, c0 + m + 1)), ctx=ctx)
        for i, e in enumerate(ents):
            st.insert_steps(c0 + i + 1, e, steps, 0)
        del ents, lat
    ids = np.arange(1, n_c + 1, dtype=np.uint64)
    ix.insert_batch(ids, ew, eo, eb)
    fill_s = time.perf_counter() - t0
    # the trace: Zipf over templates, new prompt ids, host arrays (the engine API a user calls)
    rng = np.random.default_rng(11)
    w = 1.0 / np.arange(1, 2001)
    pick = torch.as_tensor(rng.choice(2000, size=n_r, p=w / w.sum()), device=dev)
    # request noise spread so similarities cover every step bin and misses
    qw, qo, qb = (x.cpu().numpy() for x in embs(pick // 40, pick % 40,
                                              torch.rand(n_r, 1, generator=g, device=dev) * 2.0))
    lat, om, bm = make_latents(torch, n_r, F, dims, 7, dev)
    # each request's own latents arrive from pinned host memory (the e2e contract)
    lat_h, om_h, bm_h = (x.cpu().pin_memory() for x in (lat, om, bm))
    del lat
    prompts = list(range(n_c + 1, n_c + n_r + 1))
    arrivals = list(range(1, n_r + 1))
    # warm-up (untimed): one batch through a throwaway engine on the same
    # context primes one-time costs (lazy module loads, host pools) that
    # otherwise land on the first timed call (~0.1 s)
    warm = fc.Engine(cfg, ctx=ctx)
    warm.process(prompts[:64], arrivals[:64], qw[:64], qo[:64], qb[:64], lat_h[:64], om_h[:64], bm_h[:64])
    del warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs = []
    call_ms = []
    for j0 in range(0, n_r, 64):
        sl = slice(j0, j0 + 64)
        tc = time.perf_counter()
        outs += eng.process(prompts[sl], arrivals[sl], qw[sl], qo[sl], qb[sl], lat_h[sl], om_h[sl], bm_h[sl])
        call_ms.append(round((time.perf_counter() - tc) * 1e3, 2))
    if os.environ.get("FC_TRACE") == "1":
        print("[bench] engine process wall ms per call:", call_ms, file=sys.stderr)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    m = eng.metrics()
    ist = ix.stats()
    istats = {f: getattr(ist, f) for f, _ in ist._fields_}
    return {"index_stats": istats, "workload": f"config[0]: {n_c} cached prompts (768-d, 16 x 40x64x4 fp32), {n_r}-request Zipf(1.0) trace "
                        f"over a 50x40 template grid (request noise U[0,2] x per-dim sigma), LRBU, unbounded capacity, "
                        "batches of 64",
            "requests_per_s": n_r / dt, "ms_per_request": dt / n_r * 1e3, "prefill_s": fill_s,
            "whole_hits": m["whole_hits"], "decoupled_hits": m["decoupled_hits"], "misses": m["misses"],
            "skipped_hist": m["skipped_hist"], "computation_savings": m["computation_savings"],
            "throughput_vs_nocache_simulated": m["throughput_vs_nocache"],
            "api": "Engine.process (host inputs: embeddings + each prompt's latents, pinned)"}


def bench_engine_mixed(torch, fc, ctx, args, dev):
    """config[3] scaled: a cold engine serving R requests of 64-frame 40x64x4
    latents (Zipf(1.0) prompt reuse over 20,000 templates, popularity
    reshuffled every R/4 requests) under a fixed capacity budget,
    so inserts evict (LRBU) and evicted prompts leave the index. Latents are
    generated on the device per 256-request batch (generation not timed)."""
    n_r, F, dims, D = args.mixed_requests, 64, (40, 64, 4), 768
    cap = int(args.mixed_capacity_gb * (1 << 30))
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    n_t = 20000
    T = torch.randn(n_t, 3, D, generator=g, device=dev)
    cfg = fc.engine_config(dim=D, F=F, H=40, W=64, C=4, policy=int(fc.Policy.Lrbu), capacity=cap)
    eng = fc.Engine(cfg, ctx=ctx)
    rng = np.random.default_rng(21)
    w = 1.0 / np.arange(1, n_t + 1)
    w /= w.sum()
    perm = rng.permutation(n_t)
    dt, done, ev = 0.0, 0, 0
    B = 256
    for j0 in range(0, n_r, B):
        if j0 % max(B, n_r // 4) == 0 and j0:
            perm = rng.permutation(n_t)  # popularity drift
        m = min(B, n_r - j0)
        t = torch.as_tensor(perm[rng.choice(n_t, size=m, p=w)], device=dev)
        qs = []
        for k in range(3):
            raw = (T[t, k] + 0.3 * torch.rand(m, 1, generator=g, device=dev) *
                   torch.randn(m, D, generator=g, device=dev)).contiguous()
            u = torch.empty_like(raw)
            fc._check(fc.lib.lc_embedding_normalize(ctx.h, C.c_void_p(raw.data_ptr()), m, D, C.c_void_p(u.data_ptr())))
            qs.append(u.cpu().numpy())
        lat, om, bm = make_latents(torch, m, F, dims, 1000 + j0, dev)
        prompts = list(range(1 + j0, 1 + j0 + m))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = eng.process(prompts, list(range(1 + j0, 1 + j0 + m)), qs[0], qs[1], qs[2], lat, om, bm)
        torch.cuda.synchronize()
        dt += time.perf_counter() - t0
        done += m
        ev += sum(o["n_evicted"] for o in outs)
        del lat
    m_ = eng.metrics()
    return {"workload": f"config[3] scaled: {n_r} requests, 64 x 40x64x4 latents (device-resident), Zipf(1.0) over "
                        f"{n_t} templates with popularity reshuffles, LRBU, capacity {args.mixed_capacity_gb} GiB",
            "requests_per_s": done / dt, "evicted_steps": ev, "store_used_bytes": eng.store.used(),
            "whole_hits": m_["whole_hits"], "decoupled_hits": m_["decoupled_hits"], "misses": m_["misses"],
            "computation_savings": m_["computation_savings"]}


def bench_scoring(torch, fc, ctx, args, peaks):
    """Replacement scoring on a 100k-prompt x 5-step
    LRBU store (500k live steps): evict_one throughput and the scoring kernel's
    GB/s against ~53 algorithmic bytes per live step (§8(d))."""
    n_p = args.score_prompts
    steps = [5, 10, 15, 20, 25]
    F, dims = 1, (8, 8, 1)
    rng = np.random.default_rng(7)
    lat = rng.standard_normal((n_p, 5, F, 64)).astype(np.float32)
    om = np.zeros((n_p, F, 8), np.uint8)
    ents, sizes = fc.compress_batch(lat, steps, om, om, dims, list(range(1, n_p + 1)), ctx=ctx)
    st = fc.CacheStore(int(sizes.sum()) * 2, fc.Policy.Lrbu, ctx=ctx)
    t0 = time.perf_counter()
    for i, e in enumerate(ents):
        st.insert_steps(i + 1, e, steps, i + 1)
    ins_s = time.perf_counter() - t0
    del ents
    now = n_p + 1
    for pid in rng.integers(1, n_p + 1, n_p // 2):  # vary f / last_access
        st.get_step(int(pid), 25, now, want_latent=False)
        now += 1
    st.evict_one(now)  # warm-up: the first scoring uploads the whole live table (one-time, ~20 MB)
    live = st.step_count()
    fc.lib.lc_ctx_profile(ctx.h, 1)
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy", None, None, 1)
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy_call", None, None, 1)
    n_ev = args.score_evictions
    t0 = time.perf_counter()
    for _ in range(n_ev):
        st.evict_one(now)
    ev_s = time.perf_counter() - t0
    c_, t_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy", C.byref(c_), C.byref(t_), 1)
    cc_, tc_ = C.c_uint64(), C.c_double()
    fc.lib.lc_ctx_kernel_time(ctx.h, b"policy_call", C.byref(cc_), C.byref(tc_), 1)
    fc.lib.lc_ctx_profile(ctx.h, 0)
    assert st.used() == st.recompute_used()
    per_launch_ms = t_.value / c_.value if c_.value else None
    alg_bytes = live * 53
    return {"workload": f"{n_p} prompts x 5 steps LRBU, {live} live steps, {n_ev} evict_one calls",
            "evictions_per_s": n_ev / ev_s, "insert_steps_per_s": n_p / ins_s,
            "scoring_launches": int(c_.value), "scoring_ms_per_launch": per_launch_ms,
            "scoring_ms_per_call": (tc_.value / cc_.value) if cc_.value else None,
            "scoring_call_note": "call = device span from an event recorded before the host builds and issues the "
                                 "cooperative launch to the end of the report readback; it includes host launch "
                                 "latency (and any host stall in between), the kernel alone is scoring_ms_per_launch",
            "roofline": {"bound": "hbm", "kernel": "k_policy_fused (one cooperative launch: keys, radix threshold "
                                                   "select, survivor sort)",
                         "achieved": round(alg_bytes / (per_launch_ms / 1e3) / 1e9, 1) if per_launch_ms else None,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(alg_bytes / (per_launch_ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4)
                         if per_launch_ms else None,
                         "bytes_per_launch": alg_bytes, "note": "latency-bound at this size (SURVEY 8(d))"},
            "cpu_baseline": _safe(lambda: cpu_reference_evict(n_p)) if not args.no_cpu else None}


if __name__ == "__main__":
    main()
