"""GPU parity of the int8 tier-1 lookup (s8 tcgen05 shortlist with a certified
quantization bound, drop-level certificate, sorted exact rescore; bf16 tiers
and the exact scan behind it) against the restatement oracle: bit-exact ids,
fp64 scores and counts, including adversarial quantization (one-hot rows that
blow up a tile's scale), non-unit / zero queries, duplicate rows, and tiles
re-quantized by insert / remove. Reference: vindex.cpp:50-74 (query_top1
order: strict '>' over ascending ids), core.cpp:50-69 (Embedding)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def u64(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.int64 else a.astype(np.uint64)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _case(synth, n, dim, nq, seed):
    tabs = [synth.gaussian_embeddings(n, dim, seed + t) for t in range(3)]
    rng = np.random.default_rng(seed)
    nd = n // 20  # 5% exact duplicates (ties -> smaller id)
    src = rng.integers(0, n // 2, nd)
    dst = rng.integers(n // 2, n, nd)
    for t in range(3):
        tabs[t][dst] = tabs[t][src]
    ids = rng.permutation(n * 3)[:n].astype(np.uint64)
    q, _ = synth.perturbed_queries(tabs[0], nq, seed + 5)
    return tabs, ids, q


def _index(fc, tabs, ids, mode=2):
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, *tabs)
    ix.set_lookup(mode, 32)
    return ix


def _check(fc, orc, ix, tab, ids, q, k, kind=0):
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind(kind), q, k)
    oi, os_, oc = orc.topk_flat(tab, ids, q, k)
    assert (gc == oc).all()
    assert (u64(gi) == oi).all()
    assert (bits(gs) == bits(os_)).all()


@pytest.mark.parametrize("n,dim,nq,k", [
    (20000, 768, 300, 8),   # config[1] shape, ragged 256-query tiles
    (9000, 768, 257, 1),    # top-1 (query_top1), one padded query in the last pair tile
    (12000, 1024, 200, 32), # widest dim (8 K boxes in TMEM), k at the int8 tier's limit
    (5000, 128, 400, 4),    # one K box
    (3000, 384, 129, 8),    # 3 boxes (odd box count: one box per pipeline stage)
])
def test_i8_tier_exact(fc, orc, synth, n, dim, nq, k):
    tabs, ids, q = _case(synth, n, dim, nq, 3 + dim)
    ix = _index(fc, tabs, ids)
    ix.stats(reset=True)
    for kind in range(3):
        _check(fc, orc, ix, tabs[kind], ids, q, k, kind)
    s = ix.stats()
    assert s.i8_batches == 3, s.i8_batches
    assert s.certified >= 0.9 * 3 * nq, (s.certified, s.fallback)
    assert s.i8_rescored > 0


def test_i8_few_queries_use_bf16(fc, orc, synth):
    tabs, ids, q = _case(synth, 9000, 768, 100, 17)
    ix = _index(fc, tabs, ids)
    ix.stats(reset=True)
    _check(fc, orc, ix, tabs[0], ids, q, 8)
    assert ix.stats().i8_batches == 0


def test_i8_k_above_32_uses_bf16(fc, orc, synth):
    tabs, ids, q = _case(synth, 9000, 768, 200, 19)
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, *tabs)
    ix.set_lookup(2, 64)
    ix.stats(reset=True)
    _check(fc, orc, ix, tabs[0], ids, q, 40)
    assert ix.stats().i8_batches == 0


def test_i8_one_hot_rows_widen_tile_scale(fc, orc, synth):
    """A one-hot row makes its tile's scale 1/127: the other 127 rows of the
    tile quantize to a handful of levels, R8 (the max residual norm) becomes
    large and the int8 bound certifies little; the bf16 tier then answers.
    Bit-exact either way."""
    tabs, ids, q = _case(synth, 12000, 768, 300, 23)
    for t in range(3):
        for r in (5, 4000, 11999):
            tabs[t][r] = 0
            tabs[t][r][r % 768] = 1.0
    q[7] = tabs[0][4000]  # a query equal to a one-hot row: score exactly 1
    ix = _index(fc, tabs, ids)
    ix.stats(reset=True)
    for kind in range(3):
        _check(fc, orc, ix, tabs[kind], ids, q, 8, kind)
    assert ix.stats().i8_batches == 3


@pytest.mark.parametrize("scale", [3.0, 0.01, 250.0])
def test_i8_non_unit_and_zero_queries(fc, orc, synth, scale):
    tabs, ids, q = _case(synth, 10000, 768, 260, 29)
    q = (q * np.float32(scale)).astype(np.float32)
    q[3] = 0.0  # all-zero query: every score is +0.0, ids ascending
    ix = _index(fc, tabs, ids)
    _check(fc, orc, ix, tabs[0], ids, q, 8)


def test_i8_requantized_after_insert_and_remove(fc, orc, synth):
    """Inserts append into the last (partial) tile and removes move the last
    row into the hole: the touched tiles are re-quantized (scale may grow) and
    R8 only grows, so results stay exact through the mutation sequence."""
    tabs, ids, q = _case(synth, 9000, 768, 300, 31)
    ix = fc.SimilarityIndex()
    ix.set_lookup(2, 32)
    ix.insert_batch(ids[:5000], tabs[0][:5000], tabs[1][:5000], tabs[2][:5000])
    ix.insert_batch(ids[5000:5100], tabs[0][5000:5100], tabs[1][5000:5100], tabs[2][5000:5100])
    # a large-element row lands in a partial tile: that tile's scale must grow
    big = np.zeros(768, np.float32)
    big[0], big[1] = np.float32(0.8), np.float32(0.6)
    ix.insert(big, big, big, 10 ** 12)
    live = np.ones(5100, bool)
    for i in range(0, 5100, 37):
        ix.remove(int(ids[i]))
        live[i] = False
    ix.insert_batch(ids[5100:], tabs[0][5100:], tabs[1][5100:], tabs[2][5100:])
    keep = np.concatenate([live, np.ones(9000 - 5100, bool)])
    tab = np.concatenate([tabs[0][keep], big[None]])
    kid = np.concatenate([ids[keep], np.array([10 ** 12], np.uint64)])
    q2 = q.copy()
    q2[11] = big
    ix.stats(reset=True)
    _check(fc, orc, ix, tab, kid, q2, 8)
    assert ix.stats().i8_batches == 1


def test_i8_matches_bf16_tier_on_large_table(fc, synth):
    """60k rows: the int8 tier (default) and the exact scan agree bit for bit
    on 1,024 config[1]-style queries (half near-duplicates of stored rows)."""
    tabs, ids, q = _case(synth, 60000, 768, 1024, 37)
    a = _index(fc, tabs, ids, mode=2)
    a.stats(reset=True)
    ai, as_, ac = a.query_topk(fc.EmbeddingKind.Whole, q, 8)
    b = _index(fc, tabs, ids, mode=1)
    bi, bs, bc = b.query_topk(fc.EmbeddingKind.Whole, q, 8)
    assert (ai == bi).all() and (bits(as_) == bits(bs)).all() and (ac == bc).all()
    s = a.stats()
    assert s.i8_batches == 1 and s.certified >= 0.97 * 1024, (s.certified, s.fallback)
    print("i8 candidates / exact-scored per query", s.i8_candidates / 1024, s.i8_rescored / 1024)


def _clusters(n, dim, nq, csize, spread, seed):
    rng = np.random.default_rng(seed)
    base = rng.standard_normal((n, dim)).astype(np.float32)
    q = rng.standard_normal((nq, dim)).astype(np.float32)
    for j in range(nq):  # csize near-copies of each query: near-tied top-k
        base[j * csize:(j + 1) * csize] = q[j] + spread * rng.standard_normal((csize, dim)).astype(np.float32)
    perm = rng.permutation(n)
    return base[perm], q


@pytest.mark.parametrize("nq,csize", [(6, 200), (300, 150)])
def test_threshold_tier_certifies_clusters(fc, orc, nq, csize):
    """Clusters of 150-200 near-copies around each query. 6 queries (bf16
    tier first): every bf16 K' (up to 128) is inside the error bound of the
    k-th score, so they fail and the fixed-threshold int8 pass (every row with
    U above a known lower bound of T_k) certifies them. 300 queries: the int8
    tier's 256-candidate merge already holds a 150-row cluster. No fp64 scan
    either way; bit-exact with the oracle."""
    base, q = _clusters(nq * csize + 20000, 256, nq, csize, 0.01, 5 + nq)
    tab = orc.normalize_rows(base)
    qn = orc.normalize_rows(q)
    ids = (np.arange(tab.shape[0], dtype=np.uint64) * 11 + 7)
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, tab, tab, tab)
    ix.set_lookup(2, 32)
    ix.stats(reset=True)
    _check(fc, orc, ix, tab, ids, qn, 8)
    s = ix.stats()
    assert s.exact_scans == 0, s.exact_scans
    if nq <= 128:
        assert s.fallback == nq and s.threshold_certified == nq, (s.fallback, s.threshold_certified)
    else:
        assert s.i8_batches == 1 and s.certified >= 0.9 * nq, (s.certified, s.fallback)


def test_threshold_tier_off_uses_exact_scan(fc, orc):
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle');"
            "import paper_2501_04012_b200 as fc; from oracle import Checker;"
            "sys.path.insert(0, 'tests'); from test_gpu_lookup_i8 import _clusters;"
            "orc = Checker('orc'); base, q = _clusters(30000, 256, 6, 200, 0.01, 11);"
            "tab = orc.normalize_rows(base); qn = orc.normalize_rows(q);"
            "ids = np.arange(30000, dtype=np.uint64) * 3 + 1; ix = fc.SimilarityIndex();"
            "ix.insert_batch(ids, tab, tab, tab); ix.set_lookup(2, 32);"
            "gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, qn, 8); oi, os_, oc = orc.topk_flat(tab, ids, qn, 8);"
            "assert (gi.astype(np.uint64) == oi).all() and (gs == os_).all();"
            "s = ix.stats(); assert s.threshold_certified == 0 and s.exact_scans == 6, (s.threshold_certified, s.exact_scans)")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FC_LOOKUP_THRESHOLD_TIER="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_clustered_1m_table_time_and_exactness(fc, synth):
    """1M x 768 with 64 queries each surrounded by a 150-row near-tied cluster:
    bit-exact with the product's exact fp64 scan (the reference's
    sequential dot, itself pinned to the oracle), and the batch takes at most
    3x a plain (unclustered) batch of the same size -- the exact-scan
    fallback alone costs ~170 ms at this size."""
    import time
    import torch
    n, dim, nq = 1_000_000, 768, 256
    tab = synth.gaussian_embeddings(n, dim, 3)
    rng = np.random.default_rng(4)
    qc = synth.gaussian_embeddings(64, dim, 9)
    for j in range(64):
        rows = rng.choice(n, 150, replace=False)
        tab[rows] = synth.normalize_rows(qc[j] + 0.01 * rng.standard_normal((150, dim)).astype(np.float32))
    ids = np.arange(n, dtype=np.uint64)
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, tab, tab, tab)
    qp, _ = synth.perturbed_queries(tab, nq, 7)
    qcl = qp.copy()
    qcl[:64] = qc
    for qq in (qp, qcl):  # warm-up
        ix.query_topk(fc.EmbeddingKind.Whole, qq, 8)
    ts = {}
    for name, qq in (("plain", qp), ("clustered", qcl)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ix.query_topk(fc.EmbeddingKind.Whole, qq, 8)
        torch.cuda.synchronize()
        ts[name] = time.perf_counter() - t0
        if name == "clustered":
            got = res
    ex = fc.SimilarityIndex()
    ex.insert_batch(ids, tab, tab, tab)
    ex.set_lookup(1, 32)
    ei, es, ec = ex.query_topk(fc.EmbeddingKind.Whole, qcl, 8)
    assert (got[0] == ei).all() and (bits(got[1]) == bits(es)).all() and (got[2] == ec).all()
    s = ix.stats()
    print("clustered vs plain", ts, "threshold_certified", s.threshold_certified, "exact_scans", s.exact_scans)
    assert s.exact_scans == 0
    assert ts["clustered"] <= 3 * ts["plain"] + 0.005, ts
