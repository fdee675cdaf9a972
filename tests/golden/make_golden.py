"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
library (oracle/_ref/liblcache_ref.so, built from /root/reference by
oracle/Makefile). Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the plain-C restatement (oracle/lc_oracle.c) and the CUDA
product on boxes where the reference source is not available.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Checker, CheckerError, StepEntryC, build  # noqa: E402

import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location("synth", os.path.join(ROOT, "paper_2501_04012_b200", "synth.py"))
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)

DIMS = (8, 8, 4)
E = 8 * 8 * 4


def small_latents(seed, F=8, kind="synth"):
    if kind == "zero":
        return synth.zero_motion(seed, F=F, dims=DIMS)
    if kind == "norepeat":
        return synth.latents(seed, F=F, dims=DIMS, redundancy=(0, 0, 0, 0, 0))
    if kind == "prop":  # diffs exactly proportional to step 5's
        rng = np.random.default_rng(seed)
        first = rng.standard_normal(E).astype(np.float32)
        D = rng.standard_normal((F, E)).astype(np.float32)
        out = np.empty((5, F, E), np.float32)
        for i, a in enumerate((1.0, 0.9, 0.8, 0.7, 0.6)):
            out[i] = first + np.float32(a) * D
            out[i, 0] = first
        return out
    return synth.latents(seed, F=F, dims=DIMS)


def main():
    build("ref")
    ref = Checker("ref")
    kat = {}
    kat["cosine_123_456"] = ref.cosine([1, 2, 3], [4, 5, 6])
    try:
        ref.cosine([0, 0, 0], [1, 2, 3])
        kat["cosine_zero"] = "ok"
    except CheckerError as e:
        kat["cosine_zero"] = e.code
    e = StepEntryC(prompt=1, step=5, f=0, last_access=0, inserted_at=0, inserted_seq=0, capacity=1)
    kat["lrbu_unit"] = ref.lrbu(e, 1)
    e.capacity = 2
    kat["lrbu_cap2"] = ref.lrbu(e, 1)
    e2 = StepEntryC(prompt=1, step=25, f=0, capacity=7)
    kat["lcbfu_f0_s25"] = ref.lcbfu(e2)
    e3 = StepEntryC(prompt=1, step=5, f=9, capacity=7)
    kat["lcbfu_f9_s5"] = ref.lcbfu(e3)
    rng = np.random.default_rng(0)
    base = rng.standard_normal(E).astype(np.float32)
    kat["keyframes_identical"] = ref.select_keyframes(np.stack([base] * 8), DIMS).tolist()
    orth = np.zeros((8, E), np.float32)
    for j in range(8):
        orth[j, j] = 1.0
    kat["keyframes_orthogonal"] = ref.select_keyframes(orth, DIMS).tolist()
    other = rng.standard_normal(E).astype(np.float32)
    kat["keyframes_two_groups"] = ref.select_keyframes(np.stack([base] * 4 + [other] * 4), DIMS).tolist()
    # forward traversal quirk: chain A-B-C
    a = np.zeros(E, np.float32); a[0] = 1.0
    b = np.zeros(E, np.float32); b[0] = 1.0; b[1] = 0.1
    c = np.zeros(E, np.float32); c[0] = 1.0; c[1] = 0.2
    kat["keyframes_chain"] = ref.select_keyframes(np.stack([a, b, c]), DIMS).tolist()
    d = rng.standard_normal(E).astype(np.float32)
    kat["alpha_prop2"] = float(ref.solve_alpha(2 * d, d))
    try:
        ref.solve_alpha(d, np.zeros(E, np.float32))
        kat["alpha_zero_base"] = "ok"
    except CheckerError as e:
        kat["alpha_zero_base"] = e.code
    # zero-motion entry at the paper geometry
    z = synth.zero_motion(1, F=64)
    om, bm = synth.rect_masks(64, 40, 64, 1)
    zb = ref.compress(z, synth.CACHED_STEPS, om, bm, (40, 64, 4), 7)
    kat["zero_motion_size_F64"] = len(zb)
    kat["uncompressed_F64"] = 5 * 64 * 40 * 64 * 4 * 4
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)

    # ---- codec fixtures ----
    cases = [("synth", 0), ("synth", 1), ("zero", 2), ("norepeat", 3), ("prop", 4)]
    arrays = {}
    for ci, (kind, seed) in enumerate(cases):
        lat = small_latents(seed, kind=kind)
        om, bm = synth.rect_masks(8, 8, 8, seed)
        steps = np.array(synth.CACHED_STEPS, np.int32)
        if ci == 1:
            steps = steps[::-1].copy()  # unsorted input order
            lat = lat[::-1].copy()
        entry = ref.compress(lat, steps, om, bm, DIMS, 1000 + ci)
        arrays[f"c{ci}_lat"] = lat
        arrays[f"c{ci}_steps"] = steps
        arrays[f"c{ci}_om"] = om
        arrays[f"c{ci}_bm"] = bm
        arrays[f"c{ci}_entry"] = np.frombuffer(entry, np.uint8)
        for s in synth.CACHED_STEPS:
            arrays[f"c{ci}_dec{s}"] = ref.decompress(entry, s, 8, E)
        maps = np.stack([ref.select_keyframes(lat[i], DIMS) for i in range(5)])
        arrays[f"c{ci}_maps"] = maps
    # stitch toy (4x4 single channel, all 16 mask-bit combos)
    F = 1
    H, W, Cc = 4, 4, 1
    objl = np.arange(16, dtype=np.float32).reshape(1, 16) + 100
    bgl = np.arange(16, dtype=np.float32).reshape(1, 16) + 200
    bits = np.array([[(p >> 0) & 1 for p in range(16)]], bool)
    stale = np.array([[(p >> 1) & 1 for p in range(16)]], bool)
    pk = lambda m: np.packbits(m, axis=1, bitorder="little")
    arrays["stitch_obj"] = objl
    arrays["stitch_bg"] = bgl
    arrays["stitch_om"] = pk(bits)
    arrays["stitch_sm"] = pk(stale)
    arrays["stitch_out"] = ref.stitch(objl, pk(bits), pk(~bits), bgl, pk(stale), pk(~stale), (H, W, Cc))
    np.savez_compressed(os.path.join(HERE, "codec_small.npz"), **arrays)

    # ---- index fixtures ----
    dim = 64
    tabs = [synth.gaussian_embeddings(300, dim, 10 + t) for t in range(3)]
    for t in range(3):
        tabs[t][50] = tabs[t][10]  # exact duplicates -> id tie-break
        tabs[t][77] = tabs[t][10]
    ids = np.random.default_rng(5).permutation(100000)[:300].astype(np.uint64)
    ix = ref.index(dim)
    for i in range(300):
        ix.insert(int(ids[i]), tabs[0][i], tabs[1][i], tabs[2][i])
    q, _ = synth.perturbed_queries(tabs[0], 64, 6)
    q[0] = tabs[0][10]
    q[1] = tabs[1][10]
    arrays = {"ids": ids, "t0": tabs[0], "t1": tabs[1], "t2": tabs[2], "q": q}
    for k in range(3):
        i_, s_, f_ = ix.query_top1(k, q)
        arrays[f"top1_ids_{k}"] = i_
        arrays[f"top1_sc_{k}"] = s_
    np.savez_compressed(os.path.join(HERE, "index_small.npz"), **arrays)

    # ---- store sequence fixture ----
    data = np.load(os.path.join(HERE, "codec_small.npz"))
    entries = {1000 + ci: bytes(data[f"c{ci}_entry"]) for ci in range(len(cases))}
    ops = []
    rng = np.random.default_rng(9)
    for pol in range(4):
        sizes = [len(v) for v in entries.values()]
        st = ref.store(int(np.median(sizes)) * 2, pol)
        now = 0
        seq = []
        for _ in range(120):
            now += 1
            p = int(rng.choice(list(entries)))
            op = int(rng.integers(0, 3))
            if op == 0:
                steps = sorted(int(x) for x in rng.choice(synth.CACHED_STEPS, size=int(rng.integers(1, 6)),
                                                          replace=False))
                try:
                    ev = st.insert(p, entries[p], steps, now)
                    res = {"evicted": [list(map(int, e)) for e in ev]}
                except CheckerError as e:
                    res = {"error": e.code}
                seq.append({"op": "insert", "prompt": p, "steps": steps, "now": now, **res})
            elif op == 1:
                d = int(rng.choice(synth.CACHED_STEPS))
                act, _ = st.get_step(p, d, now)
                seq.append({"op": "get", "prompt": p, "desired": d, "now": now, "actual": act})
            else:
                try:
                    e = st.evict_one(now)
                    res = {"victim": list(map(int, e))}
                except CheckerError as ex:
                    res = {"error": ex.code}
                seq.append({"op": "evict", "now": now, **res})
            seq[-1]["used"] = int(st.used())
        seq.append({"op": "final", "entries": [list(map(int, e)) for e in st.entries()]})
        ops.append({"policy": pol, "capacity": int(np.median(sizes)) * 2, "seq": seq})
    with open(os.path.join(HERE, "store_seq.json"), "w") as f:
        json.dump(ops, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
