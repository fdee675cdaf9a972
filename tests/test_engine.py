"""Engine (no reference code): the SPEC's worked examples
pin the serial restatement (oracle/engine.py, CPU) and the product engine
(csrc/engine.cu, GPU); on random Zipfian traces with evictions the product
must reproduce the restatement request by request — decisions, ids, scores,
served steps, latencies, served latents (bitwise), metrics and the final
store contents."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from engine import OracleEngine, report  # noqa: E402

DIM = 32
F, DIMS = 4, (4, 4, 2)
E = DIMS[0] * DIMS[1] * DIMS[2]
MB = (DIMS[0] * DIMS[1] + 7) // 8


class World:
    """Template prompts (SPEC.md:580-598 style): object token O_i, background
    token B_k; whole = unit(O_i + B_k), object = unit(O_i), background = unit(B_k)
    (Embedding ctor rule via the C oracle, so both engines see identical bits)."""

    def __init__(self, orc, synth, n_obj=8, n_bg=6, seed=1):
        rng = np.random.default_rng(seed)
        self.O = rng.standard_normal((n_obj, DIM)).astype(np.float32)
        self.B = rng.standard_normal((n_bg, DIM)).astype(np.float32)
        self.orc, self.synth = orc, synth
        self.n_bg = n_bg

    def prompt(self, i, k):
        return 1000 + i * self.n_bg + k

    def emb(self, i, k):
        o = self.orc
        return (o.normalize(self.O[i] + self.B[k]), o.normalize(self.O[i]), o.normalize(self.B[k]))

    def latents(self, p):
        lat = self.synth.latents(p, F=F, dims=DIMS)
        om, bm = self.synth.rect_masks(F, DIMS[0], DIMS[1], p)
        return lat, om, bm

    def requests(self, n, seed, zipf=1.0):
        rng = np.random.default_rng(seed)
        n_t = len(self.O) * self.n_bg
        w = 1.0 / np.arange(1, n_t + 1) ** zipf
        pick = rng.choice(n_t, size=n, p=w / w.sum())
        out = []
        for r, t in enumerate(pick):
            i, k = divmod(int(t), self.n_bg)
            if rng.random() < 0.3:  # mixed prompt: object of one template, background of another
                k = int(rng.integers(0, self.n_bg))
            out.append((self.prompt(i, k), 10 * (r + 1), i, k))
        return out

    def arrays(self, reqs):
        qw, qo, qb, lat, om, bm = [], [], [], [], [], []
        for p, _, i, k in reqs:
            a, b, c = self.emb(i, k)
            qw.append(a), qo.append(b), qb.append(c)
            x, y, z = self.latents(p)
            lat.append(x), om.append(y), bm.append(z)
        return [np.stack(v) for v in (qw, qo, qb, lat, om, bm)]


# ---------------------------------------------------------------------------
# SPEC examples on the restatement (CPU)
# ---------------------------------------------------------------------------
def _run_oracle(eng, world, reqs):
    arr = world.arrays(reqs)
    return [eng.process(r[0], r[1], arr[0][j], arr[1][j], arr[2][j], arr[3][j], arr[4][j], arr[5][j])
            for j, r in enumerate(reqs)]


def test_spec_examples_restatement(orc, synth):
    w = World(orc, synth)
    eng = OracleEngine(orc, DIM, F, *DIMS, capacity=1 << 40)
    # cold store -> Miss, 245.74 s, 5 steps inserted
    a = _run_oracle(eng, w, [(w.prompt(0, 0), 1, 0, 0)])[0]
    assert a["kind"] == "miss" and a["n_inserted"] == 5 and abs(a["latency"] - 245.74) < 1e-9
    # identical prompt again -> WholeHit at 25, 124.74 s, nothing inserted
    b = _run_oracle(eng, w, [(w.prompt(0, 0), 2, 0, 0)])[0]
    assert b["kind"] == "whole" and b["actual_step"] == 25 and b["n_inserted"] == 0
    assert abs(b["latency"] - 124.74) < 1e-9
    m = eng.metrics()
    assert m["skipped_hist"] == {0: 1, 5: 0, 10: 0, 15: 0, 20: 0, 25: 1}
    assert m["computation_savings"] == 25 / 100
    r = report(m)
    assert abs(r["gpu_cost_per_video"] - 3.67 * (245.74 + 124.74) / 2 / 3600) < 1e-12


def test_spec_report_examples():
    # all-miss / all-hit-25 throughput and the gpu cost of one miss
    def m(lat):
        return {"requests": 1, "mean_latency": lat, "throughput_vs_nocache": 242 / lat}
    assert round(report(m(245.74))["throughput_vs_nocache"], 4) == 0.9848
    assert round(report(m(124.74))["throughput_vs_nocache"], 3) == 1.940
    assert round(report(m(245.74))["gpu_cost_per_video"], 4) == 0.2505
    with pytest.raises(ValueError):
        report({"requests": 0})


# ---------------------------------------------------------------------------
# product engine (GPU)
# ---------------------------------------------------------------------------
def _product(fc, capacity, policy=3, **kw):
    return fc.Engine(dim=DIM, F=F, H=DIMS[0], W=DIMS[1], C=DIMS[2], capacity=capacity, policy=policy, **kw)


def _cmp(a, b, j):
    for k in ("prompt", "kind", "desired_step", "actual_step", "n_inserted", "n_evicted"):
        assert a[k] == b[k], (j, k, a, b)
    assert a["latency"] == b["latency"], j
    if a["kind"] != "miss" or b["kind"] != "miss":
        assert a["score"] == b["score"], j
    # ids/scores of the three top-1s (empty index: both report miss with no ids)
    if b["scores"] != (0.0, 0.0, 0.0):
        assert (a["whole_id"], a["object_id"], a["background_id"]) == \
            (b["whole_id"], b["object_id"], b["background_id"]), j
        assert tuple(a["scores"]) == tuple(b["scores"]), j


@pytest.mark.gpu
def test_spec_examples_product(fc, orc, synth):
    w = World(orc, synth)
    eng = _product(fc, 1 << 40)
    reqs = [(w.prompt(0, 0), 1, 0, 0), (w.prompt(0, 0), 2, 0, 0)]
    arr = w.arrays(reqs)
    out = eng.process([r[0] for r in reqs], [r[1] for r in reqs], *arr)
    assert out[0]["kind"] == "miss" and out[0]["n_inserted"] == 5 and abs(out[0]["latency"] - 245.74) < 1e-9
    assert out[1]["kind"] == "whole" and out[1]["actual_step"] == 25 and abs(out[1]["latency"] - 124.74) < 1e-9
    r = eng.report()
    assert abs(r["gpu_cost_per_video"] - 3.67 * (245.74 + 124.74) / 2 / 3600) < 1e-12
    # decoupled: A holds all steps, B only {5, 10, 15} -> both served at 15
    eng2 = _product(fc, 1 << 40)
    oe = OracleEngine(orc, DIM, F, *DIMS, capacity=1 << 40)
    pa, pb = w.prompt(1, 1), w.prompt(2, 2)
    seq = [(pa, 1, 1, 1), (pb, 2, 2, 2)]
    arr = w.arrays(seq)
    eng2.process([s[0] for s in seq], [s[1] for s in seq], *arr)
    _run_oracle(oe, w, seq)
    for s in (20, 25):
        assert eng2.store.evict_step(pb, s) and oe.st.evict_step(pb, s)
    qw = orc.normalize(w.O[3] + w.B[4])  # a new whole prompt; object of A, background of B
    _, qo, _ = w.emb(1, 1)
    _, _, qb = w.emb(2, 2)
    x, om, bm = w.latents(7)
    import torch
    served = torch.zeros((1, F, E), dtype=torch.float32, device="cuda")
    got = eng2.process([7], [3], qw[None], qo[None], qb[None], x[None], om[None], bm[None], served=served)[0]
    exp = oe.process(7, 3, qw, qo, qb, x, om, bm)
    assert got["kind"] == exp["kind"] == "decoupled"
    assert got["actual_step"] == exp["actual_step"] == 15
    assert got["n_inserted"] == exp["n_inserted"] == 2  # steps 20, 25 of the new prompt
    assert (served[0].cpu().numpy().view(np.uint32) == exp["served"].view(np.uint32)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("policy,cap_prompts,batch", [(3, 1000, 1), (3, 12, 7), (0, 10, 16), (1, 9, 64),
                                                      (2, 14, 5)])
def test_random_trace_vs_restatement(fc, orc, synth, policy, cap_prompts, batch):
    import torch
    w = World(orc, synth, seed=policy + 10)
    reqs = w.requests(180, seed=policy * 7 + cap_prompts)
    lat0, om0, bm0 = w.latents(1000)
    size = len(orc.compress(lat0, (5, 10, 15, 20, 25), om0, bm0, DIMS, 1000))
    cap = size * cap_prompts
    eng = _product(fc, cap, policy)
    oe = OracleEngine(orc, DIM, F, *DIMS, capacity=cap, policy=policy)
    arr = w.arrays(reqs)
    exp = _run_oracle(oe, w, reqs)
    for j0 in range(0, len(reqs), batch):
        sl = slice(j0, j0 + batch)
        chunk = reqs[sl]
        served = torch.zeros((len(chunk), F, E), dtype=torch.float32, device="cuda")
        got = eng.process([r[0] for r in chunk], [r[1] for r in chunk], *(a[sl] for a in arr), served=served)
        sv = served.cpu().numpy()
        for t, g in enumerate(got):
            j = j0 + t
            _cmp(g, exp[j], j)
            if exp[j]["served"] is not None:
                assert (sv[t].view(np.uint32) == exp[j]["served"].view(np.uint32)).all(), j
    m, om_ = eng.metrics(), oe.metrics()
    for k in ("requests", "whole_hits", "decoupled_hits", "misses", "skipped_hist", "skipped_total",
              "simulated_time", "computation_savings", "mean_latency", "throughput_vs_nocache"):
        assert m[k] == om_[k], k
    assert m["whole_hits"] + m["decoupled_hits"] > 0 and m["misses"] > 0
    assert eng.store.used() == oe.st.used()
    assert [list(e.as_tuple()) for e in eng.store.entries_snapshot()] == [list(e) for e in oe.st.entries()]


@pytest.mark.gpu
def test_deferred_update_compress_error_leaves_no_index_orphan(fc, orc, synth):
    """A batch whose deferred (non-evicting) update cannot be compressed (a
    non-finite latent: Frame ctor, core.cpp:19-25) raises, and the prompts of
    that flush are neither in the store nor left behind in the index (a later
    lookup would otherwise hit a prompt with no data)."""
    world = World(orc, synth)
    eng = _product(fc, 1 << 40, 3)  # roomy budget: every update is deferred
    reqs = [(world.prompt(i, i % 5), 10 * (i + 1), i, i % 5) for i in range(4)]
    arr = world.arrays(reqs)
    arr[3][2, 1, 0, 5] = np.nan  # request 2's step-10 latent
    with pytest.raises(fc.InvalidArgument):
        eng.process([r[0] for r in reqs], [r[1] for r in reqs], *arr)
    ix, st = eng.index, eng.store
    for p, *_ in reqs:
        assert ix.contains(p) == st.contains(p), p
    # the engine keeps working after the failure
    reqs2 = [(world.prompt(5, 1), 100, 5, 1)]
    out = eng.process([r[0] for r in reqs2], [r[1] for r in reqs2], *world.arrays(reqs2))
    assert out[0]["kind"] == "miss" and st.contains(world.prompt(5, 1)) and ix.contains(world.prompt(5, 1))
