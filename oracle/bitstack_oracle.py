"""BitStack CPU oracle -- TEST INFRASTRUCTURE ONLY.

    Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
    `--impl reference` legs may import, call or execute anything in oracle/.
    The CUDA product path (paper_2410_23918_b200/) never imports it; the two
    share no code (the seeded generators in synthetic/ hold no method
    arithmetic).

A plain, slow, obviously-correct numpy implementation, in float64, of what the
paper (/root/reference/PAPER.md, "P:<line>") computes:

  compression   Alg.1 P:423-445  -- activation-aware scaling (Eq.3-4), then n
                iterations of absolute value decomposition (Eq.5-7)
  inference     Eq.8 P:135-138 + Eq.4 P:109-112 -- y = W_hat_n x with
                W_hat_n = (sum_{i<n} S_i (.) U_i V_i^T) diag(1/s)
  accounting    Eq.9 P:789-792 -- residual block size in bits

Orientation (reading R1): weights are [d_out, d_in] ("PyTorch"
orientation, y = W x).  The paper writes W in R^{m x n} with m = input
channels and computes X W.  So the paper's A' (Eq.5, the factor on the
m = input side) is our V [d_in, k] and B' is our U [d_out, k]; the scaling
vector s indexes input channels = columns of our W.

Every function is pinned by tests/test_oracle_*.py against something other than
itself (printed paper values, closed forms, textbook special cases, brute force
with pure-Python loops); see DESIGN.md §4 for the list.  Factor VALUES (U_i,
V_i) are "parity unpinned" across SVD implementations (R9): any
orthonormal top-k basis is correct when singular values are degenerate; only
energies, residual norms and y computed from the SAME stored blocks are pinned.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "MalformedBuffer", "LevelOutOfRange", "InvalidRank", "Block",
    "column_scaling", "scale_weight", "sign_split", "svd_topk", "rank_k_factors",
    "round_to_dtype", "bf16_bits", "pack_signs", "unpack_signs", "avd_step",
    "iavd", "compress", "restore_block", "reconstruct", "matmul_dense",
    "matmul_factored", "block_size_bits", "relative_l2",
]

STORAGE_DTYPES = ("f64", "f32", "bf16", "f16")


class MalformedBuffer(ValueError):
    """wrong length or non-zero pad bits in a packed sign buffer."""


class LevelOutOfRange(ValueError):
    """requested level outside [0, n]."""


class InvalidRank(ValueError):
    """k outside [1, min(d_out, d_in)]."""


@dataclass
class Block:
    """One residual block (Fig.3; Eq.7): packed sign matrix plus
    rank-k magnitude factors, already rounded to the storage dtype."""
    signs: np.ndarray          # uint8 [ceil(d_out*d_in/8)], canonical packing
    u: np.ndarray              # float64 [d_out, k]  (paper's B', output side)
    v: np.ndarray              # float64 [d_in, k]   (paper's A', input side)
    sigma: np.ndarray = field(default_factory=lambda: np.zeros(0))  # top-k sigma of |R|
    residual_norm_before: float = 0.0
    residual_norm_after: float = 0.0


# --------------------------------------------------------------------------
# Eq.3-4: activation-aware scaling
# --------------------------------------------------------------------------
def column_scaling(x_cal: np.ndarray, eps_rel: float = 1e-8) -> np.ndarray:
    """Eq.3: s = [||x_1||_2, ..., ||x_m||_2], the l2 norm of each
    input channel (column) of the calibration activations X in R^{p x m}.

    The paper is silent on dead channels; reading R5:
    clamp s_c >= 1e-8 * max_c s_c (or 1e-8 if all are zero) so diag(1/s) is finite.
    """
    x = np.asarray(x_cal, dtype=np.float64)
    s = np.sqrt(np.sum(x * x, axis=0))
    top = float(s.max()) if s.size else 0.0
    floor = eps_rel * top if top > 0 else eps_rel
    return np.maximum(s, floor)


def scale_weight(w: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Eq.4: X W = X diag(1/s) diag(s) W = X diag(1/s) W_scaled.

    In our [d_out, d_in] orientation the paper's diag(s) W (rows = input
    channels) is W diag(s): column c is multiplied by s_c.
    """
    w = np.asarray(w, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    if s.shape != (w.shape[1],):
        raise ValueError(f"DimensionMismatch: s {s.shape} vs W {w.shape}")
    return w * s[None, :]


# --------------------------------------------------------------------------
# Eq.1-2, Eq.5: sign split and rank-k SVD of |R|
# --------------------------------------------------------------------------
def sign_split(r: np.ndarray):
    """Eq.5: W = W_sign (.) |W|.  sign(0) = +1 (reading R6), so
    sign (.) |W| == W holds exactly for every entry."""
    r = np.asarray(r, dtype=np.float64)
    signs = np.where(r >= 0.0, 1, -1).astype(np.int8)
    return signs, np.abs(r)


def _fix_signs(a: np.ndarray, b: np.ndarray):
    """Sign convention: the largest-|entry| of each left singular
    vector is positive (ties -> lowest index); b is flipped with it."""
    for r in range(a.shape[1]):
        j = int(np.argmax(np.abs(a[:, r])))
        if a[j, r] < 0:
            a[:, r] = -a[:, r]
            b[:, r] = -b[:, r]
    return a, b


def svd_topk(m: np.ndarray, k: int, method: str = "exact", seed: int = 0,
             oversample: int = 16, power_iters: int = 4):
    """Top-k singular triplets of m (Eq.1): returns (sigma[k], a[d_out,k],
    b[d_in,k]) with m ~= a diag(sigma) b^T.

    method="exact": LAPACK (numpy.linalg.svd), a library primitive.
    method="randomized": seeded randomized subspace iteration (Halko, Martinsson
    & Tropp 2011, Alg. 4.4) with `oversample` extra columns and `power_iters`
    QR-re-orthonormalised power iterations -- used for the large shapes where
    exact SVD is too slow (SURVEY.md §8(c) "SVD method").
    """
    m = np.asarray(m, dtype=np.float64)
    d_out, d_in = m.shape
    if not (1 <= k <= min(d_out, d_in)):
        raise InvalidRank(f"k={k} outside [1, {min(d_out, d_in)}]")
    if method == "exact":
        a_full, sig, bt = np.linalg.svd(m, full_matrices=False)
        a, sig, b = a_full[:, :k].copy(), sig[:k].copy(), bt[:k, :].T.copy()
    elif method == "randomized":
        rng = np.random.default_rng(seed)
        ell = min(k + oversample, min(d_out, d_in))
        q, _ = np.linalg.qr(m @ rng.standard_normal((d_in, ell)))
        for _ in range(power_iters):
            z, _ = np.linalg.qr(m.T @ q)
            q, _ = np.linalg.qr(m @ z)
        small = q.T @ m                              # [ell, d_in]
        ua, sig, bt = np.linalg.svd(small, full_matrices=False)
        a = (q @ ua)[:, :k]
        sig = sig[:k].copy()
        b = bt[:k, :].T.copy()
    else:
        raise ValueError(method)
    a, b = _fix_signs(a, b)
    return sig, a, b


def rank_k_factors(m: np.ndarray, k: int, method: str = "exact", seed: int = 0):
    """Eq.2: W_svd = A B^T with A = [sqrt(s_1) u_1, ...],
    B = [sqrt(s_1) v_1, ...] -- the balanced sqrt(sigma) split (reading R10).
    Returns (A [d_out,k], B [d_in,k], sigma[k])."""
    sig, a, b = svd_topk(m, k, method=method, seed=seed)
    root = np.sqrt(sig)
    return a * root[None, :], b * root[None, :], sig


# --------------------------------------------------------------------------
# storage precision ("We store the singular vectors in FP16"; north star: bf16/fp32)
# --------------------------------------------------------------------------
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 -> float32 -> bfloat16 with round-to-nearest-even and
    return the raw uint16 bit patterns (reading R7: storage dtype bf16)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    lsb = (bits >> 16) & 1
    rounded = (bits + 0x7FFF + lsb) >> 16
    return (rounded & 0xFFFF).astype(np.uint16)


def _bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def round_to_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """Value of x after storage in `dtype` (returned as float64)."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "f64":
        return x.copy()
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        return _bf16_bits_to_f64(bf16_bits(x))
    raise ValueError(dtype)


# --------------------------------------------------------------------------
# sign packing (Fig.3 "packed into GPU-supported data types")
# --------------------------------------------------------------------------
def pack_signs(signs: np.ndarray) -> np.ndarray:
    """Canonical packing (reading R11; SPEC S:176-177 in [d_out,d_in] order):
    bit index j*d_in + c is element (j, c), least-significant-bit first within a
    byte, 1 = +1, 0 = -1, trailing pad bits 0.  numpy.packbits is the primitive."""
    s = np.asarray(signs)
    if not np.all((s == 1) | (s == -1)):
        raise ValueError("sign matrix must contain only +1/-1")
    return np.packbits((s.reshape(-1) > 0).astype(np.uint8), bitorder="little")


def unpack_signs(buf: np.ndarray, d_out: int, d_in: int) -> np.ndarray:
    """Inverse of pack_signs; MalformedBuffer on wrong length or
    non-zero pad bits."""
    b = np.asarray(buf, dtype=np.uint8).reshape(-1)
    nbits = d_out * d_in
    if b.size != (nbits + 7) // 8:
        raise MalformedBuffer(f"length {b.size} != ceil({nbits}/8)")
    bits = np.unpackbits(b, bitorder="little")
    if np.any(bits[nbits:]):
        raise MalformedBuffer("non-zero pad bits")
    return np.where(bits[:nbits].reshape(d_out, d_in) == 1, 1, -1).astype(np.int8)


# --------------------------------------------------------------------------
# Eq.5-8: (iterative) absolute value decomposition
# --------------------------------------------------------------------------
def avd_step(r: np.ndarray, k: int, dtype: str = "bf16", method: str = "exact",
             seed: int = 0):
    """One AVD iteration on residual R (Eq.5 P:120-125 and Eq.7):
      S = sign(R);  |R| ~= U V^T (rank-k, Eq.2 split);  round U, V to `dtype`;
      R_next = R - S (.) (U V^T)   -- with the ROUNDED factors (reading R8),
    so that the stored block is exactly what later iterations correct for.
    Returns (Block, R_next)."""
    r = np.asarray(r, dtype=np.float64)
    signs, mag = sign_split(r)
    if not np.any(mag):
        u = np.zeros((r.shape[0], k))
        v = np.zeros((r.shape[1], k))
        sig = np.zeros(k)
    else:
        u, v, sig = rank_k_factors(mag, k, method=method, seed=seed)
    u = round_to_dtype(u, dtype)
    v = round_to_dtype(v, dtype)
    r_next = r - signs * (u @ v.T)
    blk = Block(signs=pack_signs(signs), u=u, v=v, sigma=sig,
                residual_norm_before=float(np.linalg.norm(r)),
                residual_norm_after=float(np.linalg.norm(r_next)))
    return blk, r_next


def iavd(w_scaled: np.ndarray, n: int, k: int, dtype: str = "bf16",
         method: str = "exact", seed: int = 0):
    """Eq.6-8: Delta W^(i) = W - sum_{j<i} W_iavd^(j);
    W_iavd^(i) = AVD(Delta W^(i)).  Returns the n blocks in push order
    (Alg.1 P:435-437 "S.push(W^(i))")."""
    blocks = []
    r = np.asarray(w_scaled, dtype=np.float64)
    for i in range(n):
        blk, r = avd_step(r, k, dtype=dtype, method=method, seed=seed + 7919 * i)
        blocks.append(blk)
    return blocks


def compress(w: np.ndarray, x_cal: np.ndarray, n: int, k: int, dtype: str = "bf16",
             method: str = "exact", seed: int = 0):
    """Alg.1 lines 1-23 for one weight matrix: scaling once
    (Eq.3-4, applied before the loop) then n IAVD iterations.
    Returns (s [d_in], blocks)."""
    s = column_scaling(x_cal)
    return s, iavd(scale_weight(w, s), n, k, dtype=dtype, method=method, seed=seed)


def restore_block(blk: Block, d_out: int, d_in: int) -> np.ndarray:
    """W_iavd^(i) = W_sign^(i) (.) (A'_(i) B'_(i)^T)  (Eq.7)."""
    return unpack_signs(blk.signs, d_out, d_in) * (blk.u @ blk.v.T)


def reconstruct(blocks, s: np.ndarray, n: int, d_out: int, d_in: int) -> np.ndarray:
    """Dense W_hat_n = (sum_{i<n} S_i (.) U_i V_i^T) diag(1/s): Eq.8
    truncated at n blocks, mapped back through Eq.4."""
    if not (0 <= n <= len(blocks)):
        raise LevelOutOfRange(f"n={n} outside [0, {len(blocks)}]")
    acc = np.zeros((d_out, d_in))
    for blk in blocks[:n]:
        acc += restore_block(blk, d_out, d_in)
    return acc * (1.0 / np.asarray(s, dtype=np.float64))[None, :]


def matmul_dense(blocks, s: np.ndarray, n: int, x: np.ndarray) -> np.ndarray:
    """y[b, :] = W_hat_n x[b, :]  -- the dense oracle the GPU is gated against.
    x: [batch, d_in]; returns float64 [batch, d_out]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    d_out = blocks[0].u.shape[0] if blocks else 0
    w_hat = reconstruct(blocks, s, n, d_out, x.shape[1])
    return x @ w_hat.T


def matmul_factored(blocks, s: np.ndarray, n: int, x: np.ndarray) -> np.ndarray:
    """Same y from the factored formula (north star; Eq.4 + Eq.8):
    y = sum_i sum_r u_{i,r} (.) (S_i (v_{i,r} (.) (x / s))).  Brute-force cross-check."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if not (0 <= n <= len(blocks)):
        raise LevelOutOfRange(f"n={n} outside [0, {len(blocks)}]")
    d_in = x.shape[1]
    d_out = blocks[0].u.shape[0] if blocks else 0
    xs = x / np.asarray(s, dtype=np.float64)[None, :]
    y = np.zeros((x.shape[0], d_out))
    for blk in blocks[:n]:
        sm = unpack_signs(blk.signs, d_out, d_in).astype(np.float64)
        for r in range(blk.u.shape[1]):
            t = sm @ (blk.v[:, r][:, None] * xs.T)        # [d_out, batch]
            y += (blk.u[:, r][:, None] * t).T
    return y


# --------------------------------------------------------------------------
# Eq.9: residual block size
# --------------------------------------------------------------------------
def block_size_bits(m: int, n: int, k: int, factor_bits: int = 16) -> int:
    """Eq.9: delta_W = m*n + 16*k*(m+n) bits (sign bits + FP16
    singular-vector bits; reading R13: "singular values" in P:788 means vectors).
    `factor_bits`=32 gives the fp32-factor variant (reading R7)."""
    return int(m) * int(n) + int(factor_bits) * int(k) * (int(m) + int(n))


def relative_l2(y: np.ndarray, y_ref: np.ndarray) -> float:
    """Tolerance metric (reading R16): ||y - y_ref||_2 / ||y_ref||_2 per batch
    row, max over rows.  A row with y_ref == 0 must match exactly."""
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    y_ref = np.atleast_2d(np.asarray(y_ref, dtype=np.float64))
    if y.shape != y_ref.shape:
        raise ValueError(f"shape mismatch {y.shape} vs {y_ref.shape}")
    if not (np.all(np.isfinite(y)) and np.all(np.isfinite(y_ref))):
        return float("inf")          # NaN / inf never pass a tolerance
    worst = 0.0
    for a, b in zip(y, y_ref):
        nb = np.linalg.norm(b)
        if nb == 0.0:
            err = 0.0 if not np.any(a) else float("inf")
        else:
            err = float(np.linalg.norm(a - b) / nb)
        worst = max(worst, err)
    return worst
