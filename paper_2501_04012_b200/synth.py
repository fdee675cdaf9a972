"""Deterministic synthetic inputs (host side, numpy) shared by tests, smoke()
and bench.py so the reference, the restatement oracle and the CUDA path see
identical buffers.

Restates the SPEC generator behaviour (knobs
defaults.hpp:42-44): a per-step first frame, one common differential field
per key-frame index scaled by the per-step alpha schedule plus relative
Gaussian noise, a per-step redundant-frame fraction, and rectangular object
masks. simgen.cpp does not exist in the reference (simgen.hpp:46-93 is a
declaration only), so this is our own generator with the same knobs; it is
an input generator, not something the product computes.
"""
from __future__ import annotations

import numpy as np

CACHED_STEPS = (5, 10, 15, 20, 25)                    # defaults.hpp:18
REDUNDANCY = (0.9, 0.8, 0.6, 0.4, 0.25)               # defaults.hpp:42
ALPHA_SCHEDULE = (1.0, 0.9, 0.8, 0.7, 0.6)            # defaults.hpp:43
NOISE_SIGMA = 0.01                                    # defaults.hpp:44


def normalize_rows(x: np.ndarray) -> np.ndarray:
    """Embedding ctor (core.cpp:50-59) vectorised: fp64 sum of squares in
    element order, inv = 1/sqrt, (float)(v*inv).

    numpy's reductions are pairwise, so the row sums are done with an explicit
    sequential loop over columns (exactly the reference's order)."""
    x = np.ascontiguousarray(x, np.float32)
    x64 = x.astype(np.float64)
    sq = np.zeros(x.shape[0], np.float64)
    for d in range(x.shape[1]):
        sq += x64[:, d] * x64[:, d]
    inv = 1.0 / np.sqrt(sq)
    return (x64 * inv[:, None]).astype(np.float32)


def gaussian_embeddings(n: int, d: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return normalize_rows(rng.standard_normal((n, d), dtype=np.float32))


def perturbed_queries(table: np.ndarray, n: int, seed: int, hit_frac: float = 0.5,
                      dup_rows: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Config-2 query batch: hit_frac of the queries are stored rows moved by
    a random unit direction scaled by sigma ~ U[0, 1.25] (cosine spans all
    five step bins and the miss band), the rest are fresh unit Gaussians."""
    rng = np.random.default_rng(seed)
    d = table.shape[1]
    q = rng.standard_normal((n, d), dtype=np.float32)
    n_hit = int(n * hit_frac)
    src = rng.integers(0, table.shape[0], n_hit)
    u = normalize_rows(rng.standard_normal((n_hit, d), dtype=np.float32))
    sigma = rng.uniform(0.0, 1.25, n_hit).astype(np.float32)
    q[:n_hit] = table[src] + sigma[:, None] * u
    perm = rng.permutation(n)
    return normalize_rows(q[perm]), perm


def rect_masks(F: int, H: int, W: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Rectangular object masks drifting one pixel per frame; background =
    complement. Packed LSB-first per frame (core.hpp:104-124)."""
    rng = np.random.default_rng(seed)
    h0 = int(rng.integers(0, H // 2)); h1 = int(rng.integers(h0 + 1, H + 1))
    w0 = int(rng.integers(0, W // 2)); w1 = int(rng.integers(w0 + 1, W + 1))
    obj = np.zeros((F, H, W), bool)
    for j in range(F):
        s = j % max(1, W - w1 + 1)
        obj[j, h0:h1, w0 + s:min(W, w1 + s)] = True
    bg = ~obj
    pack = lambda m: np.packbits(m.reshape(F, H * W), axis=1, bitorder="little")
    return pack(obj), pack(bg)


def latents(seed: int, F: int = 16, dims=(40, 64, 4), steps=CACHED_STEPS, redundancy=REDUNDANCY,
            alphas=ALPHA_SCHEDULE, noise=NOISE_SIGMA, dup_noise: float = 0.02) -> np.ndarray:
    """[S][F][E] fp32 latents for one prompt.

    frame j of step i = first_i + alpha_i * D[j] * (1 + noise*N) for key
    frames; a redundant frame is a near-copy (relative dup_noise) of an
    earlier key frame of the same step; redundant sets nest (a frame redundant
    at a later step is redundant at every earlier one). D[j] is shared across steps so the
    inter-step differential model of codec.hpp:1-8 applies."""
    H, W, C = dims
    E = H * W * C
    rng = np.random.default_rng(seed)
    base = rng.standard_normal(E).astype(np.float32)
    D = rng.standard_normal((F, E)).astype(np.float32)
    out = np.empty((len(steps), F, E), np.float32)
    order = rng.permutation(np.arange(1, F))  # nested redundant sets across steps
    for i in range(len(steps)):
        a = alphas[i % len(alphas)]
        r = redundancy[i % len(redundancy)]
        first = base * np.float32(1.0 - 0.05 * i) + np.float32(0.05) * rng.standard_normal(E).astype(np.float32)
        n_red = int(round(r * (F - 1)))
        red = set(order[:n_red].tolist())
        keys = [0]
        out[i, 0] = first
        for j in range(1, F):
            if j in red:
                k = keys[int(rng.integers(0, len(keys)))]
                jit = rng.standard_normal(E).astype(np.float32)
                out[i, j] = out[i, k] + np.float32(dup_noise / np.sqrt(E)) * np.linalg.norm(out[i, k]) * jit
            else:
                nz = 1.0 + noise * rng.standard_normal(E).astype(np.float32)
                out[i, j] = first + np.float32(a) * D[j] * nz.astype(np.float32)
                keys.append(j)
    return out


def zero_motion(seed: int, F: int = 16, dims=(40, 64, 4), steps=CACHED_STEPS) -> np.ndarray:
    """Every frame of a step equals its first frame."""
    H, W, C = dims
    rng = np.random.default_rng(seed)
    out = np.empty((len(steps), F, H * W * C), np.float32)
    for i in range(len(steps)):
        out[i, :] = rng.standard_normal(H * W * C).astype(np.float32)
    return out
