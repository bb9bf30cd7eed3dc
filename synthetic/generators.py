"""Seeded generators for BitStack workloads (SURVEY.md §8(d) "Synthetic inputs").

Recipe (stated in DESIGN.md §3):
  * weights            W[j, c] ~ N(0, 0.02^2), shape [d_out, d_in]  (Llama-like init scale)
  * channel gains      g_c = exp(0.5 * xi_c), xi ~ N(0, 1); a seeded 0.5 % of channels
                       are x20 outliers -- "outliers ... systematically distributed
                       across the activation channels" (§2.1.1)
  * calibration        X_cal[t, c] = g_c * N(0, 1), p rows ("X in R^{p x m}")
  * decode inputs      x[b, c] = g_c * N(0, 1) with a different seed
  * seeds              1000 * config + 10 * layer + role   (role: 0 W, 1 X_cal, 2 x, 3 blocks)

`make_random_blocks` draws *already-stored-form* residual blocks (uniform random
packed sign bytes, factor matrices with IAVD-like magnitudes) for the bench:
kernel run time does not depend on the values, and bench.py's GPU leg may not
run the oracle's compression loop.  It performs none of the method's steps.
"""
from __future__ import annotations

import numpy as np

# Configurations of BASELINE.json "configs" (C1..C5); shapes are [d_out, d_in].
CONFIGS = {
    "c1": dict(d_out=256, d_in=512, n=4, k=16, batch=1, factor_dtype="f32"),
    "c2": dict(d_out=4096, d_in=4096, n=16, k=16, batch=1, factor_dtype="bf16"),
    "c3_up": dict(d_out=14336, d_in=4096, n=8, k=16, batch=2048, factor_dtype="bf16"),
    "c3_down": dict(d_out=4096, d_in=14336, n=8, k=16, batch=2048, factor_dtype="bf16"),
    "c5": dict(d_out=8192, d_in=28672, n=12, k=16, batch=1, factor_dtype="bf16"),
}

# Config C4: the paper's 8B memory points map to these average block levels per
# matrix ((budget - 2004.5 MiB embeddings/lm_head) / 912 MiB per level).
C4_LEVELS = {3674: 1.83, 3877: 2.05, 4506: 2.74, 4709: 2.97, 5338: 3.66, 5541: 3.88}


def average_levels(n_matrices: int, level: float, seed: int):
    """Per-matrix block counts for an average level ("Average" layering S:356):
    every matrix gets floor(level) blocks, and a seeded random permutation of the matrices
    receives the next block until round(frac * n_matrices) extra blocks are spent."""
    base = int(np.floor(level))
    extra = int(round((level - base) * n_matrices))
    n = np.full(n_matrices, base, np.int64)
    n[np.random.default_rng(seed).permutation(n_matrices)[:extra]] += 1
    return n


# Llama-3.1-8B per-layer linear shapes [d_out, d_in] (config C4; P:805 Table A.4 row).
LLAMA31_8B_SHAPES = {
    "q_proj": (4096, 4096),
    "k_proj": (1024, 4096),
    "v_proj": (1024, 4096),
    "o_proj": (4096, 4096),
    "gate_proj": (14336, 4096),
    "up_proj": (14336, 4096),
    "down_proj": (4096, 14336),
}

_ROLE = {"w": 0, "xcal": 1, "x": 2, "blocks": 3, "gains": 4}


def seed_for(config: int, layer: int = 0, role: str = "w") -> int:
    """Seed convention of SURVEY.md §8(d): 1000*config + 10*layer + role."""
    return 1000 * int(config) + 10 * int(layer) + _ROLE[role]


def channel_gains(d_in: int, seed: int, outlier_frac: float = 0.005,
                  outlier_gain: float = 20.0) -> np.ndarray:
    """Per-input-channel activation scale g_c (log-normal, with x20 outliers)."""
    rng = np.random.default_rng(seed)
    g = np.exp(0.5 * rng.standard_normal(d_in))
    n_out = max(1, int(round(outlier_frac * d_in)))
    idx = rng.choice(d_in, size=n_out, replace=False)
    g[idx] *= outlier_gain
    return g


def make_weight(d_out: int, d_in: int, seed: int, std: float = 0.02) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((d_out, d_in)) * std


def make_calibration(p: int, gains: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((p, gains.shape[0])) * gains[None, :]


def make_x(batch: int, gains: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, gains.shape[0])) * gains[None, :]


def random_signs_bytes(count: int, d_out: int, d_in: int, seed: int) -> np.ndarray:
    """`count` canonical packed sign buffers of uniform random bits, pad bits zero.

    Shape [count, ceil(d_out*d_in/8)] uint8.  (Uniform bytes ARE uniformly random
    packed sign matrices; only the trailing pad bits must be cleared.)
    """
    nbits = d_out * d_in
    nbytes = (nbits + 7) // 8
    rng = np.random.default_rng(seed)
    buf = rng.integers(0, 256, size=(count, nbytes), dtype=np.uint8)
    pad = nbytes * 8 - nbits
    if pad:
        buf[:, -1] &= np.uint8((1 << (8 - pad)) - 1)
    return buf


def make_random_blocks(n: int, d_out: int, d_in: int, k: int, seed: int,
                       p_cal: int = 4096):
    """Stored-form blocks for benchmarking: (signs[n, nbytes] u8, u[n,d_out,k] f32,
    v[n,d_in,k] f32, s[d_in] f32 > 0).

    Magnitudes mimic IAVD output on the synthetic recipe: s_c ~ g_c*sqrt(p),
    column 0 of u/v non-negative (Perron vector of |R|, Eq.5) and the
    residual energy roughly halving per block (802->356->180->...).
    """
    rng = np.random.default_rng(seed)
    gains = channel_gains(d_in, seed + 1)
    s = (gains * np.sqrt(p_cal)).astype(np.float32)
    signs = random_signs_bytes(n, d_out, d_in, seed + 2)
    u = np.empty((n, d_out, k), np.float32)
    v = np.empty((n, d_in, k), np.float32)
    typical = 0.02 * float(np.sqrt(p_cal))  # |R| entry scale for g=1 channels
    for i in range(n):
        amp = typical * (0.5 ** i)
        sig = amp * np.sqrt(d_out * d_in) * np.geomspace(1.0, 0.05, k)
        a = rng.standard_normal((d_out, k)) / np.sqrt(d_out)
        b = rng.standard_normal((d_in, k)) / np.sqrt(d_in)
        a[:, 0] = np.abs(a[:, 0])
        b[:, 0] = np.abs(b[:, 0])
        b *= (gains / np.sqrt(np.mean(gains ** 2)))[:, None]
        u[i] = a * np.sqrt(sig)[None, :]
        v[i] = b * np.sqrt(sig)[None, :]
    return signs, u, v, s
