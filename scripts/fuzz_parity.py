"""Randomized parity fuzzing on a B200 (developer tool, not part of the test
suite): for a fixed wall-clock budget, draws random shapes and data regimes
for the lookup (exact top-k through the certified tensor-core path, with
duplicate-heavy and near-tied tables) and the codec (compress_batch vs the
restatement oracle, byte for byte, plus decompress of every step) and stops at
the first mismatch, printing the seed to reproduce it.

  python scripts/fuzz_parity.py --minutes 10 [--seed 1]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2501_04012_b200 as fc  # noqa: E402
from paper_2501_04012_b200 import synth  # noqa: E402
from oracle import Checker  # noqa: E402


def u64(a):
    return np.ascontiguousarray(a).view(np.uint64)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.dtype == np.float64 else np.uint32)


def lookup_case(orc, rng):
    dim = int(rng.choice([64, 128, 256, 512, 768]))
    n = int(rng.choice([9000, 20000, 70000, 150000]))
    nq = int(rng.choice([1, 7, 40, 150, 300, 1000]))
    k = int(rng.choice([1, 4, 8]))
    kprime = int(rng.choice([32, 64]))
    regime = rng.choice(["random", "dups", "clusters"])
    if regime == "random":
        base = rng.standard_normal((n, dim)).astype(np.float32)
    elif regime == "dups":
        d = rng.standard_normal((max(1, n // 50), dim)).astype(np.float32)
        base = d[rng.integers(0, d.shape[0], n)]
    else:
        base = rng.standard_normal((n, dim)).astype(np.float32)
        c = rng.standard_normal((nq, dim)).astype(np.float32)
        for j in range(min(nq, n // 100)):
            base[j * 100:(j + 1) * 100] = c[j] + 0.01 * rng.standard_normal((100, dim)).astype(np.float32)
    tab = orc.normalize_rows(base)
    ids = rng.permutation(np.arange(n, dtype=np.uint64) * 3 + 1).astype(np.uint64)
    src = base[rng.integers(0, n, nq)] + 0.05 * rng.standard_normal((nq, dim)).astype(np.float32)
    q = orc.normalize_rows(src.astype(np.float32))
    ix = fc.SimilarityIndex()
    ix.insert_batch(ids, tab, tab, tab)
    ix.set_lookup(int(rng.choice([0, 2])), kprime)
    gi, gs, gc = ix.query_topk(fc.EmbeddingKind.Whole, q, k)
    oi, os_, oc = orc.topk_flat(tab, ids, q, k)
    ok = (gc == oc).all() and (u64(gi) == oi).all() and (bits(gs) == bits(os_)).all()
    return ok, f"lookup dim={dim} n={n} nq={nq} k={k} kprime={kprime} regime={regime}"


def codec_case(orc, rng):
    F = int(rng.choice([8, 13, 16, 32, 64]))
    dims = [(40, 64, 4), (8, 8, 4), (7, 9, 3), (16, 16, 4)][int(rng.integers(0, 4))]
    n = int(rng.integers(1, 6))
    S = int(rng.integers(1, 6))
    steps = rng.choice([5, 10, 15, 20, 25], size=S, replace=False).tolist()
    if rng.random() < 0.7:
        steps = sorted(steps)  # the reference sorts internally; unsorted inputs are legal too
    seed = int(rng.integers(0, 1 << 30))
    lat = np.stack([synth.latents(seed + i, F=F, dims=dims)[:S] for i in range(n)])
    if rng.random() < 0.3:  # exact duplicates / zero frames stress the select and K7 ties
        lat[:, :, F // 2] = lat[:, :, 0]
    if rng.random() < 0.2:
        lat[:, :, -1] = 0.0
    if rng.random() < 0.2:  # frames outside the tensor-core Gram's range guard [2^-40, 2^56] / denormals
        sc = float(rng.choice([1e-13, 1e-20, 1e17, 1e-41]))
        lat[int(rng.integers(0, n)), int(rng.integers(0, S)), int(rng.integers(0, F))] *= np.float32(sc)
    masks = [synth.rect_masks(F, dims[0], dims[1], seed + i) for i in range(n)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    prompts = [seed % 1000 + i for i in range(n)]
    thr = float(rng.choice([0.99, 0.95, 0.999]))
    try:
        ents, _ = fc.compress_batch(lat, steps, om, bm, dims, prompts, threshold=thr)
    except fc.InvalidArgument as ex:  # the reference must reject the batch the same way
        msgs = []
        for i in range(n):
            try:
                orc.compress(lat[i], steps, om[i], bm[i], dims, prompts[i], thr=thr)
            except Exception as ox:  # noqa: BLE001
                msgs.append(str(ox))
        return any(str(ex) in m or m in str(ex) for m in msgs), f"codec error parity: ours={ex!s} ref={msgs[:1]}"
    for i in range(n):
        want = orc.compress(lat[i], steps, om[i], bm[i], dims, prompts[i], thr=thr)
        if ents[i].serialize() != want:
            return False, f"codec compress F={F} dims={dims} S={S} steps={steps} n={n} item={i} thr={thr}"
        for si, s in enumerate(steps):
            dec = fc.decompress_step(ents[i], s)
            if not (bits(dec) == bits(orc.decompress(want, s, F, int(np.prod(dims))))).all():
                return False, f"codec decompress F={F} dims={dims} step={s} item={i}"
    return True, f"codec F={F} dims={dims} S={S} n={n}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=5.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    orc = Checker("orc")
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.minutes * 60
    n_cases = {"lookup": 0, "codec": 0}
    while time.time() < t_end:
        case_seed = int(rng.integers(0, 1 << 31))
        crng = np.random.default_rng(case_seed)
        kind = "lookup" if crng.random() < 0.5 else "codec"
        ok, desc = (lookup_case if kind == "lookup" else codec_case)(orc, crng)
        n_cases[kind] += 1
        if not ok:
            print(f"MISMATCH case_seed={case_seed}: {desc}", flush=True)
            sys.exit(1)
    print(f"fuzz ok: {n_cases['lookup']} lookup cases, {n_cases['codec']} codec cases, all bit-exact", flush=True)


if __name__ == "__main__":
    main()
