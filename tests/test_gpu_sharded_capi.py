"""GPU, world size 2 on ONE B200: the entry-sharded cache through the C-ABI
(shard.cu: lc_sharded_query_topk / lc_sharded_lookup_decide /
lc_sharded_store_*). Two processes share cuda:0; the library's collectives go
through a gloo group via the host all-gather transport (lc_ctx_comm_host),
because NCCL refuses two ranks on one device. Checked against the unsharded
CPU oracle: global top-k ids and fp64 scores, decisions, and for the store the
whole trace of insert (evicted StepEntry lists) / get_step / evict_one /
used() under one global capacity budget, including prompt ids >= 2^63."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2501_04012_b200 as fc
    from paper_2501_04012_b200 import sharded
    ctx = fc.Context(0)
    sharded.attach_comm(ctx, transport="host")
    return dist, fc, sharded, ctx


def _lookup_worker(rank, world, port, out_dir, n, d, nq, mode, skew):
    dist, fc, sharded, ctx = _init(rank, world, port)
    from oracle import Checker
    from paper_2501_04012_b200 import synth
    orc = Checker("orc")
    tabs = [synth.gaussian_embeddings(n, d, 70 + t) for t in range(3)]
    tabs[0][n - 1] = tabs[0][5]  # exact duplicates across shards: ties -> smaller id
    ids = (np.arange(n, dtype=np.uint64) * 7 + 3)
    if skew:  # rank 1 (odd ids) gets only 4,000 rows: below the tensor-core size, it scans exactly
        ids = np.arange(n, dtype=np.uint64) * 2
        ids[::n // 4000] += np.uint64(1)
    ids[:50] += np.uint64(2 ** 63)  # u64 ids above 2^63
    q = [synth.perturbed_queries(tabs[t], nq, 80 + t)[0] for t in range(3)]
    q[0][0] = tabs[0][5]
    ix = fc.SimilarityIndex(ctx=ctx)
    sh = sharded.CommShardedIndex(ix, d)
    assert sh.insert_batch(ids, *tabs) > 0
    ix.set_lookup(mode, 32)  # 2: tensor-core path on each shard; 0: by shard size
    gi, gs, gc = sh.query_topk(0, q[0], 8)
    dec = sh.lookup_decide(q[0], q[1], q[2])
    info = sharded.comm_info(ctx)
    st = ix.stats()
    res = {"fallback": st.fallback, "i8_batches": st.i8_batches, "ids": gi, "sc": gs, "cnt": gc, "dec": [(x.kind, x.step, x.whole_id, x.object_id, x.background_id,
                                                     x.score) for x in dec], "info": info}
    if rank == 0:
        oi, os_, oc = orc.topk_flat(tabs[0], ids, q[0], 8)
        top1 = [orc.topk_flat(tabs[t], ids, q[t], 1) for t in range(3)]
        ref_dec = []
        for j in range(nq):
            kind, score = orc.decide(top1[0][1][j, 0], top1[1][1][j, 0], top1[2][1][j, 0])
            ref_dec.append((kind, orc.similarity_to_step(score) if kind else 0, int(top1[0][0][j, 0]),
                            int(top1[1][0][j, 0]), int(top1[2][0][j, 0]), score))
        res["ref"] = (oi, os_, oc, ref_dec)
    with open(os.path.join(out_dir, f"l{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    del sh, ix
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,d,nq,mode,skew", [
    (20000, 256, 96, 2, False),   # bf16 tier per shard (batch too small for the int8 tier)
    (30000, 768, 300, 2, False),  # int8 tier, two-phase: shared lower bound of the global k-th score
    (30000, 768, 300, 0, True),   # one shard scans exactly, the other runs two-phase: the bound
                                  # exchange is still one collective per rank
    (72000, 768, 160, 2, False),  # shards of >= 256 row tiles: both run the pilot and filter with
                                  # the max over the ranks of the pilots' per-query keys
    (72000, 768, 160, 0, True),   # only rank 0 runs a pilot; the exact-scanning rank joins the
                                  # pilot-key exchange with -inf
])
def test_capi_sharded_lookup_two_ranks(tmp_path, n, d, nq, mode, skew):
    import torch.multiprocessing as mp
    mp.spawn(_lookup_worker, args=(2, _free_port(), str(tmp_path), n, d, nq, mode, skew), nprocs=2, join=True)
    r0 = pickle.load(open(tmp_path / "l0.pkl", "rb"))
    r1 = pickle.load(open(tmp_path / "l1.pkl", "rb"))
    oi, os_, oc, ref_dec = r0["ref"]
    for r in (r0, r1):
        assert (r["ids"].view(np.uint64) == oi).all()
        assert (r["sc"].view(np.uint64) == os_.view(np.uint64)).all()
        assert (r["cnt"] == oc).all()
        assert [x[:5] for x in r["dec"]] == [x[:5] for x in ref_dec]
        assert [x[5] for x in r["dec"]] == [x[5] for x in ref_dec]
    assert r0["info"][:3] == (2, 0, 2) and r1["info"][:3] == (2, 1, 2)
    if n >= 72000 and not skew:  # the exchanged pilot keys leave every query certified
        assert min(r0["i8_batches"], r1["i8_batches"]) >= 1 and r0["fallback"] == r1["fallback"] == 0


def _store_worker(rank, world, port, policy, id_base, batch, out_dir):
    dist, fc, sharded, ctx = _init(rank, world, port)
    from oracle import Checker
    from paper_2501_04012_b200 import synth
    orc = Checker("orc")
    rng = np.random.default_rng(policy * 7 + batch)
    dims, F = (4, 4, 2), 4
    prompts = [id_base + i for i in range(40)]
    wire = {}
    for i, p in enumerate(prompts):
        r = tuple(float(x) for x in rng.uniform(0, 1, 5))
        lat = synth.latents(1000 * policy + i, F=F, dims=dims, redundancy=r)
        om, bm = synth.rect_masks(F, 4, 4, i)
        wire[p] = orc.compress(lat, synth.CACHED_STEPS, om, bm, dims, p)
    ents = {p: fc.deserialize_entry(b, ctx=ctx) for p, b in wire.items() if int(p) % world == rank}
    sizes = sorted(len(b) for b in wire.values())
    cap = sizes[len(sizes) // 2] * 8
    ops, now = [], 0
    for _ in range(400):
        now += int(rng.integers(0, 3))
        p = int(rng.choice(prompts))
        u = rng.random()
        if u < 0.45:
            st = sorted(int(x) for x in rng.choice(synth.CACHED_STEPS, size=int(rng.integers(1, 6)), replace=False))
            ops.append(("ins", p, st, now))
        elif u < 0.85:
            ops.append(("get", p, int(rng.choice(synth.CACHED_STEPS)), now))
        else:
            ops.append(("evict", 0, 0, now))
    ss = sharded.CommShardedStore(cap, policy, ctx, batch=batch)
    ref = orc.store(cap, policy) if rank == 0 else None
    log, ref_log = [], []
    for op, p, x, now in ops:
        if op == "ins":
            try:
                got = ss.insert_steps(p, ents.get(p), x, now)
            except fc.OversizedEntry:
                got = "OversizedEntry"
            except fc.InvalidArgument:
                got = "InvalidArgument"
            log.append(got)
            if ref is not None:
                try:
                    exp = [tuple(int(v) for v in e) for e in ref.insert(p, wire[p], x, now)]
                except Exception as e:  # noqa: BLE001
                    exp = "OversizedEntry" if e.code == 4 else "InvalidArgument"
                ref_log.append(exp)
        elif op == "get":
            log.append(ss.get_step(p, x, now))
            if ref is not None:
                ref_log.append(ref.get_step(p, x, now)[0])
        else:
            try:
                log.append(ss.evict_one(now))
            except fc.LogicError:
                log.append("empty")
            if ref is not None:
                try:
                    ref_log.append(tuple(int(v) for v in ref.evict_one(now)))
                except Exception:  # noqa: BLE001
                    ref_log.append("empty")
        log.append(ss.used())
        if ref is not None:
            ref_log.append(ref.used())
    res = {"log": log, "ref": ref_log, "local_steps": ss.local.step_count() if hasattr(ss.local, "step_count") else 0,
           "stats": ss.stats()}
    with open(os.path.join(out_dir, f"s{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    del ss, ents  # library objects go before their context
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("policy,id_base,batch", [(3, 100, 64), (3, 100, 1), (0, 2 ** 63 + 100, 4), (1, 100, 64),
                                                  (2, 2 ** 64 - 41, 64)])
def test_capi_sharded_store_global_budget(tmp_path, policy, id_base, batch):
    import torch.multiprocessing as mp
    mp.spawn(_store_worker, args=(2, _free_port(), policy, id_base, batch, str(tmp_path)), nprocs=2, join=True)
    r0 = pickle.load(open(tmp_path / "s0.pkl", "rb"))
    r1 = pickle.load(open(tmp_path / "s1.pkl", "rb"))
    assert r0["log"] == r1["log"]   # every rank sees the same global outcome ...
    assert r0["log"] == r0["ref"]   # ... which is the unsharded reference-rule store's
    assert any(isinstance(x, list) and x for x in r0["log"])  # inserts did evict
    assert r0["stats"]["next_seq"] == r1["stats"]["next_seq"]
    if batch > 1:  # batched rounds: fewer collective rounds than evictions
        ev = r0["stats"]["local_evictions"] + r1["stats"]["local_evictions"]
        assert r0["stats"]["rounds"] <= ev


def _nccl_worker(port, out_dir):
    """world 1: the library's own NCCL communicator (ncclCommInitRank on
    cuda:0, dlopen'ed libnccl) drives lc_sharded_query_topk / lookup_decide,
    i.e. the collective code path the N-GPU bench uses."""
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    import paper_2501_04012_b200 as fc
    from paper_2501_04012_b200 import sharded, synth
    ctx = fc.Context(0)
    sharded.attach_comm(ctx, transport="nccl")
    nr, rk, be, _ = sharded.comm_info(ctx)
    n, d, nq, k = 20000, 256, 300, 8
    tabs = [synth.gaussian_embeddings(n, d, 90 + t) for t in range(3)]
    ids = np.arange(n, dtype=np.uint64) * 5 + 1
    q = [synth.perturbed_queries(tabs[t], nq, 95 + t)[0] for t in range(3)]
    ix = fc.SimilarityIndex(ctx=ctx)
    sh = sharded.CommShardedIndex(ix, d)
    assert sh.insert_batch(ids, *tabs) == n
    ix.set_lookup(2, 32)
    got = sh.query_topk(fc.EmbeddingKind.Whole, q[0], k)
    ref = ix.query_topk(fc.EmbeddingKind.Whole, q[0], k)
    dec = sh.lookup_decide(q[0], q[1], q[2])
    dref = fc.lookup_decide(ix, q[0], q[1], q[2])
    with open(os.path.join(out_dir, "nccl.pkl"), "wb") as f:
        pickle.dump({"comm": (nr, rk, be), "ids": (np.asarray(got[0]).view(np.uint64), np.asarray(ref[0]).view(np.uint64)),
                     "sc": (np.asarray(got[1]), np.asarray(ref[1])), "cnt": (np.asarray(got[2]), np.asarray(ref[2])),
                     "dec": ([(x.kind, x.step, x.object_id, x.background_id, x.score) for x in dec],
                             [(x.kind, x.step, x.object_id, x.background_id, x.score) for x in dref])}, f)
    dist.destroy_process_group()


def test_nccl_communicator_single_rank(tmp_path):
    import multiprocessing as mp
    ctxm = mp.get_context("spawn")
    p = ctxm.Process(target=_nccl_worker, args=(_free_port(), str(tmp_path)))
    p.start()
    p.join(600)
    assert p.exitcode == 0
    with open(tmp_path / "nccl.pkl", "rb") as f:
        r = pickle.load(f)
    assert r["comm"] == (1, 0, 1)  # one rank, backend NCCL
    for key in ("ids", "sc", "cnt"):
        a, b = r[key]
        assert (np.asarray(a) == np.asarray(b)).all(), key
    assert r["dec"][0] == r["dec"][1]
