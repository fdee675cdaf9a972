"""config[3] (and config[4] per GPU) at stated size on one B200 (diagnostic
run, not the bench):
a cold engine serves R requests (default 100,000 = 100k entries offered to the
cache) of 64-frame 4x40x64 latents with Zipf(1.0) prompt reuse over 20,000
templates (popularity reshuffled every R/4 requests) under a fixed
HBM capacity budget, so inserts evict (LRBU) and evicted prompts leave the
index (insert + lookup + evict, store.cpp:53-91 / SPEC.md:504-522).

Parity (sampled prefix): the first P requests of the same trace, at a capacity
small enough that evictions start within the prefix, run through the product
engine AND the serial CPU restatement (oracle/engine.py over the C oracle);
decisions, top-1 ids and scores, served steps, latencies, insert/evict counts,
metrics and the final store contents must be identical (bitwise).

  python scripts/config3_scale.py [--requests 100000] [--capacity-gb 16]
                                  [--prefix 400] [--prefix-capacity-gb 0.25]
config[4] per GPU (200k entries over 8 B200 = 25k offered per GPU; large
latents; per-step cache checkpoints = lc_snapshot_save of the whole store +
index every --checkpoint-every requests, timed apart from the serving):
  python scripts/config3_scale.py --dims 72x128x4 --batch 64 --requests 25000 \
      --capacity-gb 16 --checkpoint-every 5000 --prefix 96 --prefix-capacity-gb 1
Prints one JSON object (throughput + checkpoints + parity verdict).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2501_04012_b200 as fc  # noqa: E402
import bench  # noqa: E402

F, D = 64, 768
DIMS = (40, 64, 4)
N_T = 20000
B = 256


class Trace:
    """The bench_engine_mixed trace generator (bench.py), reproducible by seed."""

    def __init__(self, ctx, dev, n_r, seed=21):
        self.ctx, self.dev, self.n_r = ctx, dev, n_r
        self.g = torch.Generator(device=dev)
        self.g.manual_seed(seed)
        self.T = torch.randn(N_T, 3, D, generator=self.g, device=dev)
        self.rng = np.random.default_rng(seed)
        w = 1.0 / np.arange(1, N_T + 1)
        self.w = w / w.sum()
        self.perm = self.rng.permutation(N_T)

    def batch(self, j0, m):
        if j0 % max(B, self.n_r // 4) == 0 and j0:
            self.perm = self.rng.permutation(N_T)  # popularity drift
        t = torch.as_tensor(self.perm[self.rng.choice(N_T, size=m, p=self.w)], device=self.dev)
        qs = []
        for k in range(3):
            raw = (self.T[t, k] + 0.3 * torch.rand(m, 1, generator=self.g, device=self.dev) *
                   torch.randn(m, D, generator=self.g, device=self.dev)).contiguous()
            u = torch.empty_like(raw)
            fc._check(fc.lib.lc_embedding_normalize(self.ctx.h, C.c_void_p(raw.data_ptr()), m, D,
                                                    C.c_void_p(u.data_ptr())))
            qs.append(u.cpu().numpy())
        lat, om, bm = bench.make_latents(torch, m, F, DIMS, 1000 + j0, self.dev)
        return qs, lat, om, bm


def run_product(ctx, dev, n_r, cap, keep=0, ckpt_every=0, ckpt_dir="/dev/shm"):
    """Serve n_r requests; returns (requests/s, outcomes of the first `keep`,
    inputs of the first `keep` (host), engine, evicted steps, checkpoints)."""
    cfg = fc.engine_config(dim=D, F=F, H=DIMS[0], W=DIMS[1], C=DIMS[2], policy=int(fc.Policy.Lrbu), capacity=cap)
    eng = fc.Engine(cfg, ctx=ctx)
    tr = Trace(ctx, dev, n_r)
    dt, outs, inputs, ev, ckpts = 0.0, [], [], 0, []
    for j0 in range(0, n_r, B):
        m = min(B, n_r - j0)
        qs, lat, om, bm = tr.batch(j0, m)
        prompts = list(range(1 + j0, 1 + j0 + m))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        o = eng.process(prompts, prompts, qs[0], qs[1], qs[2], lat, om, bm)
        torch.cuda.synchronize()
        dt += time.perf_counter() - t0
        ev += sum(x["n_evicted"] for x in o)
        if j0 < keep:
            k = min(m, keep - j0)
            outs += o[:k]
            inputs.append((prompts[:k], [q[:k] for q in qs], lat[:k].cpu().numpy(), om[:k].cpu().numpy(),
                           bm[:k].cpu().numpy()))
        del lat, om, bm
        done = j0 + m
        if ckpt_every and (done % ckpt_every < B or done == n_r) and done >= ckpt_every:
            path = os.path.join(ckpt_dir, f"flexcache_ckpt_{os.getpid()}.flxc")
            t0 = time.perf_counter()
            eng.save_snapshot(path)
            sv = time.perf_counter() - t0
            sz = os.path.getsize(path)
            os.remove(path)
            ckpts.append({"after_requests": done, "bytes": sz, "save_s": round(sv, 3), "GBps": round(sz / sv / 1e9, 3)})
    return n_r / dt, outs, inputs, eng, ev, ckpts


def cmp(a, b, j):
    for k in ("prompt", "kind", "desired_step", "actual_step", "n_inserted", "n_evicted"):
        if a[k] != b[k]:
            return f"request {j}: {k} {a[k]} != {b[k]}"
    if a["latency"] != b["latency"]:
        return f"request {j}: latency"
    if (a["kind"] != "miss" or b["kind"] != "miss") and a["score"] != b["score"]:
        return f"request {j}: score"
    if b["scores"] != (0.0, 0.0, 0.0):
        if (a["whole_id"], a["object_id"], a["background_id"]) != (b["whole_id"], b["object_id"], b["background_id"]):
            return f"request {j}: top-1 ids"
        if tuple(a["scores"]) != tuple(b["scores"]):
            return f"request {j}: top-1 scores"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=100_000)
    ap.add_argument("--capacity-gb", type=float, default=16.0)
    ap.add_argument("--prefix", type=int, default=400)
    ap.add_argument("--prefix-capacity-gb", type=float, default=0.25)
    ap.add_argument("--dims", default="40x64x4")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--checkpoint-every", type=int, default=0)
    ap.add_argument("--snapshot-dir", default="/dev/shm")
    args = ap.parse_args()
    global DIMS, B
    DIMS = tuple(int(x) for x in args.dims.split("x"))
    B = args.batch
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = fc.Context(0, stream=stream.cuda_stream)
    res = {"workload": f"{args.requests} requests (entries offered), 64 x {args.dims} fp32 latents, "
                       f"768-d embeddings, Zipf(1.0) over {N_T} templates with popularity reshuffles, LRBU, "
                       f"capacity {args.capacity_gb} GiB, batches of {B}"}
    rps, _, _, eng, ev, ckpts = run_product(ctx, dev, args.requests, int(args.capacity_gb * (1 << 30)),
                                            ckpt_every=args.checkpoint_every, ckpt_dir=args.snapshot_dir)
    m = eng.metrics()
    res.update({"requests_per_s": rps, "evicted_steps": ev, "store_used_bytes": eng.store.used(),
                "live_prompts": len({e.as_tuple()[0] for e in eng.store.entries_snapshot()}),
                "whole_hits": m["whole_hits"], "decoupled_hits": m["decoupled_hits"], "misses": m["misses"],
                "computation_savings": m["computation_savings"]})
    if ckpts:
        res["checkpoints"] = {"api": "Engine.save_snapshot = lc_snapshot_save (FLXC v1, byte-identical to the "
                                     "reference's save_snapshot, store.cpp:232-274), whole store + index",
                              "target": args.snapshot_dir, "runs": ckpts}
    del eng
    # ---- parity on the prefix (same trace, small capacity so evictions start early) ----
    if args.prefix > 0:
        from oracle import Checker
        from engine import OracleEngine
        orc = Checker("orc")
        cap = int(args.prefix_capacity_gb * (1 << 30))
        _, outs, inputs, eng, ev, _ = run_product(ctx, dev, args.prefix, cap, keep=args.prefix)
        oe = OracleEngine(orc, D, F, *DIMS, capacity=cap, policy=int(fc.Policy.Lrbu))
        t0 = time.perf_counter()
        exp, j, bad = [], 0, None
        for prompts, qs, lat, om, bm in inputs:
            for t, p in enumerate(prompts):
                exp.append(oe.process(p, p, qs[0][t], qs[1][t], qs[2][t], lat[t], om[t], bm[t]))
        cpu_s = time.perf_counter() - t0
        for j, (a, b) in enumerate(zip(outs, exp)):
            bad = cmp(a, b, j)
            if bad:
                break
        pm, om_ = eng.metrics(), oe.metrics()
        if not bad:
            for k in ("requests", "whole_hits", "decoupled_hits", "misses", "skipped_hist", "skipped_total",
                      "simulated_time", "computation_savings"):
                if pm[k] != om_[k]:
                    bad = f"metric {k}"
                    break
        if not bad and eng.store.used() != oe.st.used():
            bad = "store bytes"
        if not bad and [list(e.as_tuple()) for e in eng.store.entries_snapshot()] != [list(e) for e in oe.st.entries()]:
            bad = "store entries"
        res["parity_prefix"] = {"requests": len(exp), "capacity_gb": args.prefix_capacity_gb, "evicted_steps": ev,
                                "misses": om_["misses"], "whole_hits": om_["whole_hits"],
                                "decoupled_hits": om_["decoupled_hits"], "identical": bad is None,
                                "first_difference": bad, "oracle_cpu_s": round(cpu_s, 1),
                                "compared": "kind, desired/actual step, inserted/evicted, latency, score, top-1 ids "
                                            "and scores per request; metrics; final store bytes and entries"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
