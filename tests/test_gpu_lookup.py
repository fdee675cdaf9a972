"""GPU parity: SimilarityIndex lookup (exact scan and the tcgen05 shortlist +
fp64 rescore + certification path) against the restatement oracle and the
reference-generated golden top-1 vectors. Bit-exact ids and fp64 scores."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def u64(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.int64 else a.astype(np.uint64)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def build_index(fc, tabs, ids, mode=0, kprime=0):
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, tabs[0], tabs[1], tabs[2])
    ix.set_lookup(mode, kprime)
    return ix


@pytest.mark.parametrize("mode", [1, 2])
def test_golden_top1(fc, mode):
    z = np.load(os.path.join(GOLD, "index_small.npz"))
    ix = build_index(fc, [z["t0"], z["t1"], z["t2"]], z["ids"], mode=mode)
    for k in range(3):
        ids, sc, cnt = ix.query_topk(fc.EmbeddingKind(k), z["q"], 1)
        assert (cnt == 1).all()
        assert (u64(ids[:, 0]) == z[f"top1_ids_{k}"]).all()
        assert (bits(sc[:, 0]) == bits(z[f"top1_sc_{k}"])).all()
    r = ix.query_top1(fc.EmbeddingKind.Whole, z["q"][0])
    assert r.prompt == int(z["top1_ids_0"][0])


def _random_case(synth, n_rows, dim, nq, seed, dups=True):
    tabs = [synth.gaussian_embeddings(n_rows, dim, seed + t) for t in range(3)]
    rng = np.random.default_rng(seed)
    if dups:  # 5% exact duplicates of earlier rows (ties -> smaller id)
        nd = max(1, n_rows // 20)
        src = rng.integers(0, n_rows // 2, nd)
        dst = rng.integers(n_rows // 2, n_rows, nd)
        for t in range(3):
            tabs[t][dst] = tabs[t][src]
    ids = rng.permutation(n_rows * 4)[:n_rows].astype(np.uint64)
    q, _ = synth.perturbed_queries(tabs[0], nq, seed + 99)
    return tabs, ids, q


@pytest.mark.parametrize("n_rows,dim,nq,k", [(3000, 768, 40, 8), (1000, 64, 17, 3)])
def test_exact_scan_topk_vs_oracle(fc, orc, synth, n_rows, dim, nq, k):
    tabs, ids, q = _random_case(synth, n_rows, dim, nq, 7)
    ix = build_index(fc, tabs, ids, mode=1)
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, q, k)
    oi, os_, oc = orc.topk_flat(tabs[0], ids, q, k)
    assert (gc == oc).all()
    assert (u64(gi) == oi).all()
    assert (bits(gs) == bits(os_)).all()


@pytest.mark.parametrize("n_rows,dim,nq,k,kp", [
    (20000, 768, 300, 8, 64),    # BN=64 path, multi-split, ragged query tile
    (9000, 512, 130, 8, 32),     # BN=128 path, kprime 32
    (5000, 256, 64, 1, 64),
    (777, 128, 5, 4, 128),       # tiny table: rows < splits*64, ragged last tile
    (40, 64, 3, 8, 64),          # fewer rows than the shortlist
])
def test_tensor_core_path_is_exact(fc, orc, synth, n_rows, dim, nq, k, kp):
    tabs, ids, q = _random_case(synth, n_rows, dim, nq, 11 + dim)
    ix = build_index(fc, tabs, ids, mode=2, kprime=kp)
    ix.stats(reset=True)
    for kind in range(3):
        gi, gs, gc = ix.query_topk(fc.EmbeddingKind(kind), q, k)
        oi, os_, oc = orc.topk_flat(tabs[kind], ids, q, k)
        assert (gc == oc).all()
        assert (u64(gi) == oi).all(), kind
        assert (bits(gs) == bits(os_)).all(), kind
    s = ix.stats()
    assert s.queries == 3 * nq
    assert s.certified + s.fallback == 3 * nq
    assert s.max_abs_err < 2 ** -8, s.max_abs_err  # measured bf16 error under the certified bound


def test_tensor_core_vs_exact_mode_large(fc, synth):
    tabs, ids, q = _random_case(synth, 60000, 768, 512, 5)
    a = build_index(fc, tabs, ids, mode=2)
    a.stats(reset=True)
    ai, as_, ac = a.query_topk(fc.EmbeddingKind.Whole, q, 8)
    b = build_index(fc, tabs, ids, mode=1)
    bi, bs, bc = b.query_topk(fc.EmbeddingKind.Whole, q, 8)
    assert (ai == bi).all() and (bits(as_) == bits(bs)).all() and (ac == bc).all()
    s = a.stats()
    print("certified", s.certified, "fallback", s.fallback, "max_err", s.max_abs_err)
    assert s.certified >= 0.9 * 512


def test_device_tensors_in_place(fc, synth):
    import torch
    tabs, ids, q = _random_case(synth, 9000, 768, 256, 3)
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, *(torch.from_numpy(t).cuda() for t in tabs))
    qd = torch.from_numpy(q).cuda()
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Object, qd, 8)
    assert gi.is_cuda
    hi, hs, hc = ix.query_topk(fc.EmbeddingKind.Object, q, 8)
    assert (u64(gi.cpu().numpy()) == hi).all() and (gs.cpu().numpy() == hs).all()


def test_insert_remove_contains_export(fc, orc, synth):
    tabs, ids, q = _random_case(synth, 500, 64, 10, 21, dups=False)
    ix = fc.SimilarityIndex()
    oix = orc.index(64)
    for i in range(500):
        ix.insert(tabs[0][i], tabs[1][i], tabs[2][i], int(ids[i]))
        oix.insert(int(ids[i]), tabs[0][i], tabs[1][i], tabs[2][i])
    with pytest.raises(fc.InvalidArgument):
        ix.insert(tabs[0][0], tabs[1][0], tabs[2][0], int(ids[0]))
    with pytest.raises(fc.InvalidArgument):
        ix.insert(tabs[0][0][:32], tabs[1][0][:32], tabs[2][0][:32], 10 ** 9)
    with pytest.raises(fc.InvalidArgument):  # not unit norm (from_unit, core.cpp:66)
        ix.insert(tabs[0][0] * 2, tabs[1][0], tabs[2][0], 10 ** 9)
    for i in range(0, 500, 3):
        ix.remove(int(ids[i]))
        oix.remove(int(ids[i]))
    with pytest.raises(fc.InvalidArgument):
        ix.remove(int(ids[0]))
    assert ix.size() == oix.size()
    assert ix.contains(int(ids[1])) and not ix.contains(int(ids[0]))
    for kind in range(3):
        eid, rows = ix.entries(fc.EmbeddingKind(kind))
        assert (np.diff(eid.astype(np.int64)) > 0).all()
        r_ids, r_sc, r_f = oix.query_top1(kind, q)
        res = [ix.query_top1(fc.EmbeddingKind(kind), qq) for qq in q]
        assert [r.prompt for r in res] == r_ids.tolist()
        assert [r.score for r in res] == r_sc.tolist()


def test_empty_index(fc):
    ix = fc.SimilarityIndex(dim=64)
    assert ix.query_top1(fc.EmbeddingKind.Whole, np.ones(64, np.float32) / 8) is None
    d = fc.lookup_decide(ix, *(np.ones((2, 64), np.float32) / 8,) * 3)
    assert d[0].kind == 0 and d[1].kind == 0


def test_lookup_decide_vs_oracle(fc, orc, synth):
    tabs, ids, q = _random_case(synth, 12000, 768, 200, 31)
    rng = np.random.default_rng(3)
    qo, _ = synth.perturbed_queries(tabs[1], 200, 5)
    qb, _ = synth.perturbed_queries(tabs[2], 200, 6)
    ix = build_index(fc, tabs, ids)
    dec = fc.lookup_decide(ix, q, qo, qb)
    res = []
    for t, qq in enumerate((q, qo, qb)):
        oi, os_, oc = orc.topk_flat(tabs[t], ids, qq, 1)
        res.append((oi[:, 0], os_[:, 0]))
    kinds = [0, 0, 0]
    for i in range(200):
        kind, score = orc.decide(res[0][1][i], res[1][1][i], res[2][1][i])
        assert dec[i].kind == kind
        assert dec[i].score == score
        assert dec[i].whole_id == res[0][0][i] and dec[i].object_id == res[1][0][i]
        if kind:
            assert dec[i].step == orc.similarity_to_step(score)
        kinds[kind] += 1
    assert min(kinds) > 0, kinds  # all three outcomes exercised


def test_topk_merge_equals_unsharded(fc, orc, synth):
    tabs, ids, q = _random_case(synth, 4000, 64, 50, 41)
    G, k = 4, 8
    shard = (ids % G).astype(int)
    gi = np.zeros((G, 50, k), np.uint64)
    gs = np.zeros((G, 50, k))
    gc = np.zeros((G, 50), np.int32)
    for g in range(G):
        m = shard == g
        gi[g], gs[g], gc[g] = orc.topk_flat(tabs[0][m], ids[m], q, k)
    mi, ms, mc = fc.topk_merge(gi, gs, gc, k)
    oi, os_, oc = orc.topk_flat(tabs[0], ids, q, k)
    assert (mi == oi).all() and (bits(ms) == bits(os_)).all() and (mc == oc).all()


def test_sharded_index_product_path_single_rank(fc, orc, synth):
    """paper_2501_04012_b200.sharded on the GPU: a world-size-1 NCCL group with
    the device index, packed all-gather and lc_topk_merge on device tensors;
    plus G=3 logical shards (id mod 3) merged on the device — both equal the
    unsharded oracle bit for bit (the multi-rank host logic is covered by the
    gloo tests in test_sharded.py)."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2501_04012_b200 import sharded
    tabs, ids, q = _random_case(synth, 12000, 768, 64, 23)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ix = fc.SimilarityIndex()
        sh = sharded.ShardedIndex(ix)
        assert sh.insert_batch(ids, *tabs) == len(ids)
        qd = torch.from_numpy(q).cuda()
        gi, gs, gc = sh.query_topk(0, qd, 8)
        oi, os_, oc = orc.topk_flat(tabs[0], ids, q, 8)
        assert (u64(gi.cpu().numpy()) == oi).all() and (bits(gs.cpu().numpy()) == bits(os_)).all()
        assert (gc.cpu().numpy() == oc).all()
        dec = sh.lookup_decide(qd, qd, qd)
        ref = fc.lookup_decide(ix, q, q, q)
        assert [(d.kind, d.step, d.whole_id) for d in dec] == [(d.kind, d.step, d.whole_id) for d in ref]
    finally:
        dist.destroy_process_group()
    # G = 3 logical shards on one GPU, merged on the device
    G = 3
    parts = []
    for g in range(G):
        m = sharded.owner_of(ids, G) == np.uint64(g)
        ixg = fc.SimilarityIndex()
        ixg.insert_batch(ids[m], tabs[0][m], tabs[1][m], tabs[2][m])
        parts.append(ixg.query_topk(fc.EmbeddingKind.Whole, torch.from_numpy(q).cuda(), 8))
    mi, ms, mc = fc.topk_merge(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]),
                               torch.stack([p[2] for p in parts]), 8)
    assert (u64(mi.cpu().numpy()) == oi).all() and (bits(ms.cpu().numpy()) == bits(os_)).all()


@pytest.mark.parametrize("tier2", ["1", "0"])
def test_near_tied_cluster_tier2_and_exact(fc, orc, synth, tier2):
    """100 rows within ~1e-3 of each other around each query: the K'=32 bf16
    shortlist cannot certify the top-8 (its 32nd score is inside the error
    bound of the 8th), the K'=128 re-shortlist can; with FC_LOOKUP_TIER2=0 the
    exact scan answers. Both are bit-exact with the oracle."""
    os.environ["FC_LOOKUP_TIER2"] = tier2
    try:
        rng = np.random.default_rng(41)
        n, dim, nq = 20000, 256, 6
        base = rng.standard_normal((n, dim)).astype(np.float32)
        q = rng.standard_normal((nq, dim)).astype(np.float32)
        for j in range(nq):  # a cluster of 100 near-copies of each query
            for c in range(100):
                base[j * 100 + c] = q[j] + 0.01 * rng.standard_normal(dim).astype(np.float32)
        tab = orc.normalize_rows(base)
        qn = orc.normalize_rows(q)
        ids = np.arange(n, dtype=np.uint64) * 7 + 3
        ix = build_index(fc, [tab, tab, tab], ids, mode=2, kprime=32)
        ix.stats(reset=True)
        gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, qn, 8)
        oi, os_, oc = orc.topk_flat(tab, ids, qn, 8)
        assert (u64(gi) == oi).all() and (bits(gs) == bits(os_)).all() and (gc == oc).all()
        s = ix.stats()
        assert s.fallback == nq, s.fallback
        if tier2 == "1":
            assert s.tier2_certified == nq and s.exact_scans == 0, (s.tier2_certified, s.exact_scans)
        else:
            assert s.tier2_certified == 0
    finally:
        del os.environ["FC_LOOKUP_TIER2"]


@pytest.mark.parametrize("nq", [40, 300])
def test_duplicate_heavy_table_merge_paths(fc, orc, nq):
    """A table of 1,000 distinct rows each stored 100 times (100k rows): every
    work unit's shortlist fills up with equal scores, so the per-query merge
    sees more filled slots than its shared-memory buffer (global spill path,
    nq >= the SM count) or runs one CTA per query (nq < the SM count); ties
    are broken by id exactly as the oracle does, and the uncertifiable queries
    take the exact scan. Bit-exact with the oracle either way."""
    rng = np.random.default_rng(77)
    dim = 64
    distinct = orc.normalize_rows(rng.standard_normal((1000, dim)).astype(np.float32))
    tab = np.repeat(distinct, 100, axis=0)
    perm = rng.permutation(tab.shape[0])
    tab = np.ascontiguousarray(tab[perm])
    ids = (np.arange(tab.shape[0], dtype=np.uint64) * 13 + 5)
    q = orc.normalize_rows((distinct[rng.integers(0, 1000, nq)] +
                            0.05 * rng.standard_normal((nq, dim))).astype(np.float32))
    ix = build_index(fc, [tab, tab, tab], ids, mode=2, kprime=32)
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, q, 8)
    oi, os_, oc = orc.topk_flat(tab, ids, q, 8)
    assert (gc == oc).all()
    assert (u64(gi) == oi).all() and (bits(gs) == bits(os_)).all()


def _cluster_case(orc, seed, n=20000, dim=256, nq=6, spread=0.01):
    rng = np.random.default_rng(seed)
    base = rng.standard_normal((n, dim)).astype(np.float32)
    q = rng.standard_normal((nq, dim)).astype(np.float32)
    for j in range(nq):  # 100 near-copies of each query: near-tied top-8s
        for c in range(100):
            base[j * 100 + c] = q[j] + spread * rng.standard_normal(dim).astype(np.float32)
    return orc.normalize_rows(base), orc.normalize_rows(q)


@pytest.mark.parametrize("scale", [8.0, 100.0, 0.125])
def test_non_unit_queries_stay_exact(fc, orc, scale):
    """The C-ABI takes raw floats, so a caller can pass queries that are not
    unit (the reference cannot: queries are Embeddings, core.cpp:50-69). The
    certified bound scales with ||q|| (k_rescore), so a query of norm 8 or 100
    near a cluster of near-ties must still return the exact top-8 of the
    sequential fp64 dot (vindex.cpp:66-67), bit for bit."""
    tab, qn = _cluster_case(orc, 91, spread=0.03)
    ids = np.arange(tab.shape[0], dtype=np.uint64) * 5 + 1
    q = (qn * np.float32(scale)).astype(np.float32)
    ix = build_index(fc, [tab, tab, tab], ids, mode=2, kprime=32)
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, q, 8)
    oi, os_, oc = orc.topk_flat(tab, ids, q, 8)
    assert (u64(gi) == oi).all() and (bits(gs) == bits(os_)).all() and (gc == oc).all()


@pytest.mark.parametrize("mode", [1, 2])
def test_non_finite_query_rejected(fc, synth, mode):
    tabs, ids, q = _random_case(synth, 9000, 256, 40, 13)
    ix = build_index(fc, tabs, ids, mode=mode)
    q = q.copy()
    q[17, 3] = np.nan
    with pytest.raises(fc.InvalidArgument):
        ix.query_topk(fc.EmbeddingKind.Whole, q, 8)
    q[17, 3] = np.inf
    with pytest.raises(fc.InvalidArgument):
        ix.query_topk(fc.EmbeddingKind.Whole, q, 8)
    q[17, 3] = 0.0
    ix.query_topk(fc.EmbeddingKind.Whole, q, 8)  # finite again: accepted


def test_eps_below_proven_bound_is_clamped(fc, orc):
    """lc_index_set_lookup cannot make the certificate unsound: an eps below
    2^-8 + 2^-12 is raised to it, so near-tied clusters (which the bf16
    shortlist cannot certify) still end bit-exact."""
    tab, qn = _cluster_case(orc, 41)
    ids = np.arange(tab.shape[0], dtype=np.uint64) * 7 + 3
    ix = build_index(fc, [tab, tab, tab], ids, mode=2, kprime=32)
    ix.set_lookup(2, 32, 1e-12)
    ix.stats(reset=True)
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, qn, 8)
    oi, os_, oc = orc.topk_flat(tab, ids, qn, 8)
    assert (u64(gi) == oi).all() and (bits(gs) == bits(os_)).all() and (gc == oc).all()
    assert ix.stats().fallback == qn.shape[0]
