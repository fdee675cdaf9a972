"""GPU parity: latent codec (select_keyframes, solve_alpha, compress =
intra x S + inter, wire format, decompress, stitch, fused decompress+stitch)
against the reference golden fixtures and the restatement oracle.
Integer/byte outputs and decompressed floats are compared bit-for-bit."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIMS = (8, 8, 4)
E = 256


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32)


def test_golden_entries(fc):
    z = np.load(os.path.join(GOLD, "codec_small.npz"))
    ci = 0
    while f"c{ci}_lat" in z:
        ent = fc.compress(z[f"c{ci}_lat"], z[f"c{ci}_steps"], z[f"c{ci}_om"], z[f"c{ci}_bm"], DIMS, 1000 + ci)
        wire = ent.serialize()
        assert wire == bytes(z[f"c{ci}_entry"]), f"case {ci}"
        assert fc.compressed_size(ent) == len(wire)
        for s in (5, 10, 15, 20, 25):
            assert (bits(fc.decompress_step(ent, s)) == bits(z[f"c{ci}_dec{s}"])).all()
        maps = fc.select_keyframes(z[f"c{ci}_lat"], DIMS)
        assert (maps == z[f"c{ci}_maps"]).all()
        ci += 1


@pytest.mark.parametrize("F,dims,seed", [(16, (40, 64, 4), 0), (64, (40, 64, 4), 1), (13, (7, 9, 3), 2)])
def test_compress_batch_vs_oracle(fc, orc, synth, F, dims, seed):
    n = 3
    lat = np.stack([synth.latents(seed * 10 + i, F=F, dims=dims) for i in range(n)])
    masks = [synth.rect_masks(F, dims[0], dims[1], seed * 10 + i) for i in range(n)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    prompts = [500 + i for i in range(n)]
    ents, sizes = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, prompts)
    E_ = dims[0] * dims[1] * dims[2]
    for i in range(n):
        ref_bytes = orc.compress(lat[i], synth.CACHED_STEPS, om[i], bm[i], dims, prompts[i])
        assert ents[i].serialize() == ref_bytes
        assert int(sizes[i]) == len(ref_bytes)
        for s in synth.CACHED_STEPS:
            assert (bits(fc.decompress_step(ents[i], s)) == bits(orc.decompress(ref_bytes, s, F, E_))).all()


def test_edge_latents(fc, orc, synth):
    dims = (40, 64, 4)
    for lat in (synth.zero_motion(3, F=64), synth.latents(4, F=16, redundancy=(0, 0, 0, 0, 0)),
                synth.latents(5, F=16, redundancy=(1, 1, 1, 1, 1))):
        F = lat.shape[1]
        om, bm = synth.rect_masks(F, 40, 64, 1)
        ent = fc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 9)
        assert ent.serialize() == orc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 9)
    z = synth.zero_motion(1, F=64)
    om, bm = synth.rect_masks(64, 40, 64, 1)
    ent = fc.compress(z, synth.CACHED_STEPS, om, bm, dims, 7)
    assert fc.compressed_size(ent) == 246435  # SPEC.md:202 zero-motion ratio 53.19
    for s in synth.CACHED_STEPS:  # every frame bit-exact
        dec = fc.decompress_step(ent, s)
        assert (bits(dec) == bits(z[synth.CACHED_STEPS.index(s)])).all()


def test_subset_and_single_step(fc, orc, synth):
    dims = (16, 16, 4)
    lat = synth.latents(8, F=12, dims=dims)
    om, bm = synth.rect_masks(12, 16, 16, 8)
    for steps, rows in (([10], [1]), ([25, 5, 15], [4, 0, 2])):
        ent = fc.compress(lat[rows], steps, om, bm, dims, 3)
        assert ent.serialize() == orc.compress(lat[rows], steps, om, bm, dims, 3)


def test_errors(fc, synth):
    dims = (8, 8, 4)
    lat = synth.latents(3, F=4, dims=dims)
    om, bm = synth.rect_masks(4, 8, 8, 3)
    bad = lat.copy()
    bad[1, 2, 5] = np.inf
    with pytest.raises(fc.InvalidArgument):
        fc.compress(bad, synth.CACHED_STEPS, om, bm, dims, 1)
    zero = lat.copy()
    zero[2, 1] = 0
    with pytest.raises(fc.InvalidArgument):
        fc.compress(zero, synth.CACHED_STEPS, om, bm, dims, 1)
    with pytest.raises(fc.InvalidArgument):
        fc.compress(lat, (5, 5, 10, 15, 20), om, bm, dims, 1)
    with pytest.raises(fc.InvalidArgument):
        fc.select_keyframes(lat[0], dims, threshold=0.0)
    ent = fc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 1)
    with pytest.raises(fc.StepNotCached):
        fc.decompress_step(ent, 7)
    wire = ent.serialize()
    for cut in (5, 40, len(wire) - 1):
        with pytest.raises(fc.SnapshotError):
            fc.deserialize_entry(wire[:cut])
    with pytest.raises(fc.DegenerateBase):
        fc.solve_alpha(np.ones(10, np.float32), np.zeros(10, np.float32))


def test_wire_roundtrip(fc, synth):
    dims = (40, 64, 4)
    lat = synth.latents(12, F=16)
    om, bm = synth.rect_masks(16, 40, 64, 12)
    ent = fc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 42)
    wire = ent.serialize()
    back = fc.deserialize_entry(wire)
    assert back.serialize() == wire
    for s in synth.CACHED_STEPS:
        assert (bits(fc.decompress_step(back, s)) == bits(fc.decompress_step(ent, s))).all()


def test_solve_alpha_and_cosine(fc, orc):
    rng = np.random.default_rng(1)
    ds = rng.standard_normal((20, 5000)).astype(np.float32)
    db = rng.standard_normal((20, 5000)).astype(np.float32)
    ga = fc.solve_alpha(ds, db)
    oa = np.array([orc.solve_alpha(ds[i], db[i]) for i in range(20)], np.float32)
    assert (bits(ga) == bits(oa)).all()
    gc = fc.cosine_similarity(ds, db)
    oc = np.array([orc.cosine(ds[i], db[i]) for i in range(20)])
    assert (gc.view(np.uint64) == oc.view(np.uint64)).all()
    v = rng.standard_normal((50, 768)).astype(np.float32)
    assert (bits(fc.embedding_normalize(v)) == bits(orc.normalize_rows(v))).all()


def test_stitch_golden_and_random(fc, orc, synth):
    z = np.load(os.path.join(GOLD, "codec_small.npz"))
    out = fc.stitch(z["stitch_obj"], z["stitch_om"], z["stitch_bg"], z["stitch_sm"], (4, 4, 1))
    assert (bits(out) == bits(z["stitch_out"])).all()
    dims = (40, 64, 4)
    a = synth.latents(1, F=16)[2]
    b = synth.latents(2, F=16)[2]
    oo, ob = synth.rect_masks(16, 40, 64, 1)
    bo, bb = synth.rect_masks(16, 40, 64, 2)
    g = fc.stitch(a, oo, b, bo, dims)
    o = orc.stitch(a, oo, ob, b, bo, bb, dims)
    assert (bits(g) == bits(o)).all()
    assert (bits(fc.stitch(a, oo, a, oo, dims)) == bits(a)).all()  # idempotence


def test_decompress_stitch_fused(fc, orc, synth):
    dims = (40, 64, 4)
    F = 16
    la, lb = synth.latents(21, F=F), synth.latents(22, F=F)
    ma, mb = synth.rect_masks(F, 40, 64, 21), synth.rect_masks(F, 40, 64, 22)
    ea = fc.compress(la, synth.CACHED_STEPS, ma[0], ma[1], dims, 1)
    eb = fc.compress(lb, synth.CACHED_STEPS, mb[0], mb[1], dims, 2)
    wa, wb = ea.serialize(), eb.serialize()
    E_ = 40 * 64 * 4
    for s in (5, 15, 25):
        fused = fc.decompress_stitch([ea], [eb], [s])[0].cpu().numpy()
        da, db = orc.decompress(wa, s, F, E_), orc.decompress(wb, s, F, E_)
        ref = orc.stitch(da, ma[0], ma[1], db, mb[0], mb[1], dims)
        assert (bits(fused) == bits(ref)).all()


def test_inter_compress_with_maps(fc, orc, synth):
    dims = (40, 64, 4)
    lat = synth.latents(30, F=16)
    om, bm = synth.rect_masks(16, 40, 64, 30)
    maps = fc.select_keyframes(lat, dims)
    ent = fc.inter_compress(lat, maps, synth.CACHED_STEPS, om, bm, dims, 99)
    assert ent.serialize() == orc.compress(lat, synth.CACHED_STEPS, om, bm, dims, 99)


def _near_threshold_latent(rng, F, E, thr=0.99):
    """Frames whose cosine to an earlier key sits within the tensor-core Gram's
    certified bound (1e-4) of the threshold, and frames equally similar to two
    keys (argmax ties broken by the reference's fp64 rounding), so
    k_select_cert must fall back to exact sequential fp64 dots."""
    unit = lambda v: v / np.linalg.norm(v)
    x = np.zeros((F, E), np.float32)
    k0 = unit(rng.standard_normal(E))
    x[0] = k0 * 3.0
    offs = [-3e-5, -1e-5, -2e-6, 0.0, 2e-6, 1e-5, 3e-5, 9e-5]
    j = 1
    for d in offs:  # sim(j, 0) = thr + d (up to fp32 rounding of the frame)
        c = thr + d
        u = unit(rng.standard_normal(E) - (rng.standard_normal(E) @ k0) * k0)
        u = unit(u - (u @ k0) * k0)
        x[j] = (c * k0 + np.sqrt(1 - c * c) * u) * (1.0 + 0.1 * j)
        j += 1
    # two keys 0.985 apart and their bisector (sim ~0.9962 to both)
    a = unit(rng.standard_normal(E))
    b = unit(0.985 * a + np.sqrt(1 - 0.985 ** 2) * unit(rng.standard_normal(E)))
    x[j] = a; j += 1
    x[j] = b; j += 1
    x[j] = unit(a + b) * 2.0; j += 1
    while j < F:
        x[j] = unit(rng.standard_normal(E)) * 0.5
        j += 1
    return x


def test_certified_select_near_threshold_and_ties(fc, orc):
    """tcgen05 Gram + certified select against the oracle on adversarial
    latents, and the tensor-core path against the exact-Gram path."""
    dims = (40, 64, 4)
    E_ = 40 * 64 * 4
    rng = np.random.default_rng(123)
    F = 16
    lats = np.stack([_near_threshold_latent(rng, F, E_) for _ in range(6)])
    got = fc.select_keyframes(lats, dims)
    for i in range(lats.shape[0]):
        ref = orc.select_keyframes(lats[i], dims)
        assert (got[i] == ref).all(), (i, got[i], ref)
    # the same through compress (5 steps = perturbations of the same frames)
    steps = [5, 10, 15, 20, 25]
    lat5 = np.stack([np.stack([lats[i] * np.float32(1 + 0.01 * s) for s in range(5)]) for i in range(2)])
    om = np.zeros((2, F, 40 * 64 // 8), np.uint8)
    ents, sizes = fc.compress_batch(lat5, steps, om, om, dims, [31, 32])
    for i in range(2):
        assert ents[i].serialize() == orc.compress(lat5[i], steps, om[i], om[i], dims, 31 + i)


def test_tensor_core_gram_equals_exact_gram_path(fc, synth):
    """FC_GRAM_EXACT=1 forces the sequential-fp64 Gram kernel; maps and wire
    bytes must not depend on which Gram produced them."""
    dims = (40, 64, 4)
    lat = np.stack([synth.latents(70 + i, F=64, dims=dims) for i in range(2)])
    masks = [synth.rect_masks(64, 40, 64, 70 + i) for i in range(2)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    a, _ = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, [1, 2])
    os.environ["FC_GRAM_EXACT"] = "1"
    try:
        b, _ = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, [1, 2])
    finally:
        del os.environ["FC_GRAM_EXACT"]
    for x, y in zip(a, b):
        assert x.serialize() == y.serialize()


def test_certified_inter_equals_exact_path(fc, orc, synth):
    """The certified K7 (reassociated sums + bounds) must give the same
    entries as the sequential-fp64 K7 (FC_INTER_EXACT=1) and the oracle; on
    the synthetic generator every item is settled without the exact kernel."""
    dims = (40, 64, 4)
    n = 6
    lat = np.stack([synth.latents(90 + i, F=64, dims=dims) for i in range(n)])
    masks = [synth.rect_masks(64, 40, 64, 90 + i) for i in range(n)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    fc.codec_stats(reset=True)
    a, sa = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, list(range(n)))
    st = fc.codec_stats(reset=True)
    assert st["inter_items"] > 0 and st["inter_exact_items"] == 0, st
    os.environ["FC_INTER_EXACT"] = "1"
    try:
        b, sb = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, list(range(n)))
    finally:
        del os.environ["FC_INTER_EXACT"]
    assert fc.codec_stats()["inter_exact_items"] == st["inter_items"]
    for i, (x, y) in enumerate(zip(a, b)):
        assert x.serialize() == y.serialize()
    # every alpha through the in-kernel sequential chain replay
    os.environ["FC_INTER_REPLAY"] = "1"
    try:
        c, _ = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, list(range(n)))
    finally:
        del os.environ["FC_INTER_REPLAY"]
    for x, y in zip(a, c):
        assert x.serialize() == y.serialize()
    for i in (0, n - 1):
        assert a[i].serialize() == orc.compress(lat[i], synth.CACHED_STEPS, om[i], bm[i], dims, i)


def test_certified_inter_ties_fall_back(fc, orc, synth):
    """Steps that are exact copies make every trial base score identical (the
    reference keeps the first by strict '>'); the bounds cannot separate
    them, so those prompts must go through the exact kernel. Mixed with
    ordinary prompts in one batch."""
    dims = (40, 64, 4)
    F = 16
    one = synth.latents(7, F=F, dims=dims)
    tie = np.stack([one[0]] * 5)                     # five identical steps
    tie2 = np.stack([one[0] * np.float32(1.0 + 2.0 ** -20 * s) for s in range(5)])  # near-identical
    lat = np.stack([synth.latents(8, F=F, dims=dims), tie, tie2])
    om, bm = synth.rect_masks(F, 40, 64, 8)
    om = np.stack([om] * 3)
    bm = np.stack([bm] * 3)
    fc.codec_stats(reset=True)
    ents, _ = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, [1, 2, 3])
    st = fc.codec_stats(reset=True)
    assert st["inter_exact_items"] > 0, st
    for i in range(3):
        assert ents[i].serialize() == orc.compress(lat[i], synth.CACHED_STEPS, om[i], bm[i], dims, i + 1), i


def test_large_latent_shape_config4(fc, orc, synth):
    """config[4] geometry: 64 frames of 72x128x4 (576x1024 video latents):
    tensor-core Gram path (E = 36,864), certified K7, decompress and the
    fused decoupled stitch stay bit-exact with the oracle."""
    dims = (72, 128, 4)
    F = 64
    n = 2
    lat = np.stack([synth.latents(300 + i, F=F, dims=dims) for i in range(n)])
    masks = [synth.rect_masks(F, 72, 128, 300 + i) for i in range(n)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    ents, sizes = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, [1, 2])
    E_ = 72 * 128 * 4
    for i in range(n):
        ref = orc.compress(lat[i], synth.CACHED_STEPS, om[i], bm[i], dims, i + 1)
        assert ents[i].serialize() == ref
        assert (bits(fc.decompress_step(ents[i], 15)) == bits(orc.decompress(ref, 15, F, E_))).all()
    fused = fc.decompress_stitch([ents[0]], [ents[1]], [20])[0].cpu().numpy()
    da = orc.decompress(ents[0].serialize(), 20, F, E_)
    db = orc.decompress(ents[1].serialize(), 20, F, E_)
    exp = orc.stitch(da, om[0], bm[0], db, om[1], bm[1], dims)
    assert (bits(fused) == bits(exp)).all()


def test_gram_range_guard_and_denormals(fc, orc, synth):
    """The tensor-core Gram's error model holds for frames whose max |x| lies in
    [2^-40, 2^56] (gram_sm100.cu); items with a frame outside (tiny or huge
    scales, all-denormal frames) must take select's exact path, and denormal
    elements must not be mistaken for zeros (zero-norm rule, core.cpp:111-112).
    Wire bytes equal the restatement's in every case."""
    dims = (8, 8, 4)
    F = 16
    n = 4
    lat = np.stack([synth.latents(300 + i, F=F, dims=dims) for i in range(n)]).astype(np.float32)
    lat[0, 1] *= np.float32(1e-13)             # a whole step below 2^-40
    lat[1, 2, 5] *= np.float32(1e17)           # one frame above 2^56
    lat[2, 3, 7, :5] = np.float32(1e-40)       # denormal elements in a normal frame
    lat[3, 4, 3] = (lat[3, 4, 3] * np.float32(1e-41)).astype(np.float32)  # an all-denormal (nonzero) frame
    assert np.all(lat[3, 4, 3][lat[3, 4, 3] != 0] < 1.2e-38)
    masks = [synth.rect_masks(F, dims[0], dims[1], 300 + i) for i in range(n)]
    om = np.stack([m[0] for m in masks])
    bm = np.stack([m[1] for m in masks])
    prompts = [40 + i for i in range(n)]
    ents, _ = fc.compress_batch(lat, synth.CACHED_STEPS, om, bm, dims, prompts)
    for i in range(n):
        assert ents[i].serialize() == orc.compress(lat[i], synth.CACHED_STEPS, om[i], bm[i], dims, prompts[i]), i
