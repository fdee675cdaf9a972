"""simgen (the reference declares it but ships no code).
CPU: the restatement (oracle/lc_oracle.c orc_synth_*) satisfies the SPEC's
stated properties. GPU: csrc/simgen.cu reproduces the restatement bit for bit."""
import numpy as np
import pytest

DIMS = (8, 16, 4)


def test_embedding_properties(orc):
    rng = np.random.default_rng(0)
    a = orc.synth_embedding([1, 2, 3], 512, 7)
    assert float(a @ orc.synth_embedding([1, 2, 3], 512, 7)) == pytest.approx(1.0, abs=1e-6)
    assert abs(float(np.linalg.norm(a.astype(np.float64))) - 1.0) < 1e-6  # from_unit holds (core.cpp:61-69)
    small = 0
    for t in range(300):  # disjoint token sets, dim 512: |sim| < 0.2 w.p. > 0.99
        x = orc.synth_embedding(rng.integers(0, 1 << 60, 3), 512, t)
        y = orc.synth_embedding(rng.integers(0, 1 << 60, 3), 512, t)
        small += abs(float(x @ y)) < 0.2
    assert small >= 297
    for t in range(100):  # supersets: sim(A, A u B) > sim(A, C)
        A, B, Cc = (list(rng.integers(0, 1 << 60, 2)) for _ in range(3))
        ea = orc.synth_embedding(A, 256, t)
        assert float(ea @ orc.synth_embedding(A + B, 256, t)) > float(ea @ orc.synth_embedding(Cc, 256, t))


def test_latent_redundancy_knob_is_faithful(orc):
    """noise 0 and exact duplicates: select_keyframes at 0.99 keeps exactly
    F - round(r (F-1)) key frames per step; noise 0:
    solve_alpha recovers the alpha schedule."""
    F = 32
    for seed in (1, 2, 3):
        lat, om, bm = orc.synth_latents(seed, F, DIMS, noise=0.0, dup=0.0)
        for i, r in enumerate((0.9, 0.8, 0.6, 0.4, 0.25)):
            keys = (orc.select_keyframes(lat[i], DIMS) == np.arange(F)).sum()
            assert keys == F - int(np.floor(r * (F - 1) + 0.5)), (seed, i)
        # a frame that is a key in every step (redundancy nests) recovers alpha_i / alpha_0
        maps = [orc.select_keyframes(lat[i], DIMS) for i in range(5)]
        common = [j for j in range(1, F) if all(m[j] == j for m in maps)]
        assert common
        j = common[0]
        d0 = lat[0, j] - lat[0, 0]
        for i, a in enumerate((1.0, 0.9, 0.8, 0.7, 0.6)):
            di = lat[i, j] - lat[i, 0]
            assert float(orc.solve_alpha(di, d0)) == pytest.approx(a, rel=1e-5)
        assert om.shape == (F, (DIMS[0] * DIMS[1] + 7) // 8) and ((om & bm) == 0).all()


@pytest.mark.gpu
def test_gpu_simgen_matches_restatement(fc, orc):
    rng = np.random.default_rng(3)
    sets = [list(rng.integers(0, 1 << 62, int(rng.integers(1, 6)))) for _ in range(64)]
    got = fc.synth_embeddings(sets, 768, 99).cpu().numpy()
    for i, t in enumerate(sets):
        assert (got[i].view(np.uint32) == orc.synth_embedding(t, 768, 99).view(np.uint32)).all(), i
    seeds = [5, 17, 1 << 40]
    for F, dims in ((16, DIMS), (64, (40, 64, 4))):
        lat, om, bm = fc.synth_latents(seeds, F, dims)
        lat, om, bm = lat.cpu().numpy(), om.cpu().numpy(), bm.cpu().numpy()
        for i, s in enumerate(seeds):
            el, eo, eb = orc.synth_latents(s, F, dims)
            assert (lat[i].view(np.uint32) == el.view(np.uint32)).all(), (F, i)
            assert (om[i] == eo).all() and (bm[i] == eb).all()
    # the generated latents are valid codec inputs: compress matches the oracle
    lat, om, bm = fc.synth_latents([21], 16, (40, 64, 4))
    ent = fc.compress(lat[0], [5, 10, 15, 20, 25], om[0], bm[0], (40, 64, 4), 21)
    assert ent.serialize() == orc.compress(lat[0].cpu().numpy(), [5, 10, 15, 20, 25], om[0].cpu().numpy(),
                                           bm[0].cpu().numpy(), (40, 64, 4), 21)
