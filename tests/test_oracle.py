"""CPU: the plain-C restatement (oracle/lc_oracle.c) against the golden
fixtures generated from the reference library and, when the reference was
built here, against the reference itself on fresh random inputs."""
import json
import os

import numpy as np
import pytest

from oracle import CheckerError, StepEntryC

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIMS = (8, 8, 4)
E = 256


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32 if a.dtype == np.float32 else np.uint64)


def test_kat(orc):
    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    assert orc.cosine([1, 2, 3], [4, 5, 6]) == kat["cosine_123_456"]
    with pytest.raises(CheckerError) as ei:
        orc.cosine([0, 0, 0], [1, 2, 3])
    assert ei.value.code == kat["cosine_zero"]
    e = StepEntryC(prompt=1, step=5, f=0, capacity=1)
    assert orc.lrbu(e, 1) == kat["lrbu_unit"] == 5.0
    e.capacity = 2
    assert orc.lrbu(e, 1) == kat["lrbu_cap2"]
    assert orc.lcbfu(StepEntryC(step=25, f=0, capacity=1)) == kat["lcbfu_f0_s25"] == 25
    assert orc.lcbfu(StepEntryC(step=5, f=9, capacity=1)) == kat["lcbfu_f9_s5"] == 50
    rng = np.random.default_rng(0)
    base = rng.standard_normal(E).astype(np.float32)
    assert orc.select_keyframes(np.stack([base] * 8), DIMS).tolist() == kat["keyframes_identical"]
    orth = np.zeros((8, E), np.float32)
    for j in range(8):
        orth[j, j] = 1
    assert orc.select_keyframes(orth, DIMS).tolist() == kat["keyframes_orthogonal"]
    other = rng.standard_normal(E).astype(np.float32)
    assert orc.select_keyframes(np.stack([base] * 4 + [other] * 4), DIMS).tolist() == kat["keyframes_two_groups"]
    a = np.zeros(E, np.float32); a[0] = 1
    b = np.zeros(E, np.float32); b[0] = 1; b[1] = 0.1
    c = np.zeros(E, np.float32); c[0] = 1; c[1] = 0.2
    assert orc.select_keyframes(np.stack([a, b, c]), DIMS).tolist() == kat["keyframes_chain"] == [0, 0, 2]
    d = rng.standard_normal(E).astype(np.float32)
    assert float(orc.solve_alpha(2 * d, d)) == kat["alpha_prop2"] == 2.0
    with pytest.raises(CheckerError) as ei:
        orc.solve_alpha(d, np.zeros(E, np.float32))
    assert ei.value.code == kat["alpha_zero_base"]


def test_decide_rule(orc):
    # SPEC.md:490-502 examples
    assert orc.decide(0.90, 0.70, 0.70) == (1, 0.90)
    assert orc.decide(0.60, 0.80, 0.90) == (2, 0.80)
    assert orc.decide(0.60, 0.90, 0.60)[0] == 0
    assert orc.similarity_to_step(0.65) == 5
    assert orc.similarity_to_step(0.80) == 15
    assert orc.similarity_to_step(1.0) == 25
    # 21^3 grid against an independent restatement, ties included
    g = np.round(np.linspace(0, 1, 21), 2)
    for w in g:
        for o in g:
            for b in g:
                m = min(o, b)
                exp = 0 if max(w, m) < 0.65 else (2 if (m > w and m >= 0.65) else 1)
                assert orc.decide(w, o, b)[0] == exp


def test_codec_golden(orc):
    z = np.load(os.path.join(GOLD, "codec_small.npz"))
    ci = 0
    while f"c{ci}_lat" in z:
        entry = orc.compress(z[f"c{ci}_lat"], z[f"c{ci}_steps"], z[f"c{ci}_om"], z[f"c{ci}_bm"], DIMS, 1000 + ci)
        assert entry == bytes(z[f"c{ci}_entry"]), f"case {ci}: entry bytes differ from reference"
        for s in (5, 10, 15, 20, 25):
            dec = orc.decompress(entry, s, 8, E)
            assert (bits(dec) == bits(z[f"c{ci}_dec{s}"])).all()
        for i in range(5):
            assert (orc.select_keyframes(z[f"c{ci}_lat"][i], DIMS) == z[f"c{ci}_maps"][i]).all()
        ci += 1
    out = orc.stitch(z["stitch_obj"], z["stitch_om"], ~z["stitch_om"], z["stitch_bg"], z["stitch_sm"],
                     ~z["stitch_sm"], (4, 4, 1))
    assert (bits(out) == bits(z["stitch_out"])).all()


def test_index_golden(orc):
    z = np.load(os.path.join(GOLD, "index_small.npz"))
    ix = orc.index(64)
    for i in range(300):
        ix.insert(int(z["ids"][i]), z["t0"][i], z["t1"][i], z["t2"][i])
    for k in range(3):
        ids, sc, fd = ix.query_top1(k, z["q"])
        assert (ids == z[f"top1_ids_{k}"]).all()
        assert (bits(sc) == bits(z[f"top1_sc_{k}"])).all()
        # top-k generalisation agrees with top-1 and is sorted (score desc, id asc)
        ti, ts, tc = orc.topk_flat(z[f"t{k}"], z["ids"], z["q"], 8)
        assert (ti[:, 0] == ids).all()
        for r in range(ts.shape[0]):
            for j in range(7):
                assert ts[r, j] > ts[r, j + 1] or (ts[r, j] == ts[r, j + 1] and ti[r, j] < ti[r, j + 1])
    # duplicates: the smaller id wins
    ids, sc, fd = ix.query_top1(0, z["q"][:1])
    dup = sorted(int(z["ids"][i]) for i in (10, 50, 77))
    assert int(ids[0]) == dup[0]
    e = orc.index(64)
    ids, sc, fd = e.query_top1(0, z["q"][:2])
    assert (fd == 0).all()


def test_store_golden(orc):
    z = np.load(os.path.join(GOLD, "codec_small.npz"))
    entries = {}
    ci = 0
    while f"c{ci}_entry" in z:
        entries[1000 + ci] = bytes(z[f"c{ci}_entry"])
        ci += 1
    for case in json.load(open(os.path.join(GOLD, "store_seq.json"))):
        st = orc.store(case["capacity"], case["policy"])
        for op in case["seq"]:
            if op["op"] == "insert":
                try:
                    ev = st.insert(op["prompt"], entries[op["prompt"]], op["steps"], op["now"])
                    assert "error" not in op, op
                    assert [list(e) for e in ev] == op["evicted"]
                except CheckerError as e:
                    assert op.get("error") == e.code
            elif op["op"] == "get":
                act, _ = st.get_step(op["prompt"], op["desired"], op["now"])
                assert act == op["actual"]
            elif op["op"] == "evict":
                try:
                    assert list(st.evict_one(op["now"])) == op["victim"]
                except CheckerError as e:
                    assert op.get("error") == e.code
            else:
                assert [list(e) for e in st.entries()] == op["entries"]
                continue
            assert st.used() == op["used"] == st.recompute_used()


@pytest.mark.parametrize("seed", range(4))
def test_restatement_vs_reference_codec(orc, ref, synth, seed):
    F = 16 if seed < 2 else 12
    dims = (8, 16, 4) if seed % 2 else (6, 10, 3)
    lat = synth.latents(100 + seed, F=F, dims=dims)
    om, bm = synth.rect_masks(F, dims[0], dims[1], seed)
    steps = list(synth.CACHED_STEPS)[: 5 - seed % 3]
    lat = lat[: len(steps)]
    a = ref.compress(lat, steps, om, bm, dims, 77 + seed)
    b = orc.compress(lat, steps, om, bm, dims, 77 + seed)
    assert a == b
    E_ = dims[0] * dims[1] * dims[2]
    for s in steps:
        assert (bits(ref.decompress(a, s, F, E_)) == bits(orc.decompress(a, s, F, E_))).all()
    assert ref.entry_info(a) == orc.entry_info(a)


def test_restatement_vs_reference_errors(orc, ref, synth):
    lat = synth.latents(3, F=4, dims=DIMS)
    om, bm = synth.rect_masks(4, 8, 8, 3)
    bad = lat.copy()
    bad[1, 2, 5] = np.inf
    zero = lat.copy()
    zero[2, 1] = 0
    for x, steps in ((bad, synth.CACHED_STEPS), (zero, synth.CACHED_STEPS), (lat, (5, 5, 10, 15, 20)),
                     (lat, (0, 5, 10, 15, 20))):
        codes = []
        for chk in (ref, orc):
            try:
                chk.compress(x, steps, om, bm, DIMS, 1)
                codes.append(0)
            except CheckerError as e:
                codes.append(e.code)
        assert codes[0] == codes[1] != 0
    entry = ref.compress(lat, synth.CACHED_STEPS, om, bm, DIMS, 1)
    for cut in (5, 40, len(entry) - 1):
        c1 = c2 = 0
        try:
            ref.decompress(entry[:cut], 5, 4, E)
        except CheckerError as e:
            c1 = e.code
        try:
            orc.decompress(entry[:cut], 5, 4, E)
        except CheckerError as e:
            c2 = e.code
        assert c1 == c2 == 5
    for chk in (ref, orc):
        with pytest.raises(CheckerError) as ei:
            chk.decompress(entry, 7, 4, E)
        assert ei.value.code == 3
