"""Pins of the CPU oracle against things other than itself.

Each test names the passage it pins and the plausible mistake it would catch.
"""
import itertools
import os
from decimal import ROUND_HALF_UP, Decimal

import numpy as np
import pytest

from oracle import bitstack_oracle as O
from synthetic import channel_gains, make_calibration, make_weight, make_x
from bitstack_test_helpers import read_golden


# ---------------------------------------------------------------- Eq.9 / Table A.4
def test_table_a4_block_sizes(golden_dir):
    """P1: Eq.9 reproduces every printed entry of Table A.4."""
    rows = read_golden(os.path.join(golden_dir, "table_a4.txt"))
    assert len(rows) == 35
    for model, matrix, m, n, printed in rows:
        mib = Decimal(O.block_size_bits(int(m), int(n), 16)) / Decimal(8 * 2 ** 20)
        assert mib.quantize(Decimal("0.01"), rounding=ROUND_HALF_UP) == Decimal(printed), \
            (model, matrix, mib)


def test_block_size_spec_examples():
    """SPEC S:398-400, S:424 (bits and bytes of single blocks)."""
    assert O.block_size_bits(4096, 4096, 16) == 18_874_368
    assert O.block_size_bits(4096, 1024, 16) == 5_505_024
    assert O.block_size_bits(4096, 11008, 16) == 48_955_392
    assert O.block_size_bits(4096, 4096, 16) // 8 == 2_359_296
    # A dropped factor term or a swapped coefficient would break this closed form:
    assert O.block_size_bits(3, 5, 2) == 15 + 16 * 2 * 8
    assert O.block_size_bits(3, 5, 2, factor_bits=32) == 15 + 32 * 2 * 8


# ---------------------------------------------------------------- Eq.3-4
def test_column_scaling_examples():
    """Eq.3: s_c = ||X[:, c]||_2.  SPEC S:119-120 examples."""
    np.testing.assert_array_equal(O.column_scaling(np.eye(2)), [1.0, 1.0])
    s = O.column_scaling(np.array([[3.0, 0.0], [4.0, 0.0]]))
    assert s[0] == 5.0 and s[1] == pytest.approx(5e-8, rel=1e-12)   # clamp (reading R5)


def test_column_scaling_brute_force():
    """Norm per COLUMN (input channel), not per row: pure-Python loop oracle."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((16, 8))
    want = [sum(x[t, c] ** 2 for t in range(16)) ** 0.5 for c in range(8)]
    np.testing.assert_allclose(O.column_scaling(x), want, rtol=1e-12)


def test_scaled_inference_identity_eq4():
    """Eq.4: X W = X diag(1/s) W_scaled.  In [d_out,d_in] orientation the
    scale multiplies columns of W; scaling rows instead fails this."""
    rng = np.random.default_rng(11)
    w = rng.standard_normal((5, 4))
    s = rng.uniform(0.1, 3.0, 4)
    x = rng.standard_normal((3, 4))
    ws = O.scale_weight(w, s)
    np.testing.assert_allclose((x / s) @ ws.T, x @ w.T, rtol=1e-12, atol=1e-12)
    # and the literal SPEC example S:138: s = ones -> plain product
    np.testing.assert_array_equal(O.scale_weight(w, np.ones(4)), w)
    with pytest.raises(ValueError):
        O.scale_weight(w, np.ones(5))


# ---------------------------------------------------------------- Eq.1-2
def test_svd_special_cases():
    """SPEC S:50, S:59 (diag(3,2)); Eq.2 balanced sqrt(sigma) split."""
    m = np.diag([3.0, 2.0])
    sig, a, b = O.svd_topk(m, 2)
    np.testing.assert_allclose(sig, [3.0, 2.0])
    np.testing.assert_allclose(np.abs(a), np.eye(2), atol=1e-15)
    A, B, _ = O.rank_k_factors(m, 1)
    np.testing.assert_allclose(A[:, 0], [np.sqrt(3.0), 0.0], atol=1e-15)
    np.testing.assert_allclose(B[:, 0], [np.sqrt(3.0), 0.0], atol=1e-15)
    with pytest.raises(O.InvalidRank):
        O.svd_topk(m, 3)


def test_eckart_young_against_eigen_oracle():
    """||M - A B^T||_F = sqrt(sigma_3^2 + sigma_4^2) for k=2, with
    sigma taken from an independent eigen-solver of M^T M (not numpy.linalg.svd)."""
    rng = np.random.default_rng(7)
    m = rng.standard_normal((6, 4))
    A, B, _ = O.rank_k_factors(m, 2)
    ev = np.sort(np.linalg.eigvalsh(m.T @ m))[::-1]
    assert np.linalg.norm(m - A @ B.T) == pytest.approx(np.sqrt(ev[2] + ev[3]), rel=1e-10)
    assert np.linalg.norm(np.array([[3.0, 4.0]])) == 5.0


def test_randomized_svd_energy_matches_exact():
    """The seeded randomized top-k (used at large shapes) captures the exact energy."""
    rng = np.random.default_rng(5)
    m = np.abs(rng.standard_normal((300, 200)))
    s_exact, _, _ = O.svd_topk(m, 16, method="exact")
    s_rand, a, b = O.svd_topk(m, 16, method="randomized", seed=1)
    # |Gaussian| has a Perron value then a near-flat bulk (SURVEY finding 7), so
    # the subspace iteration converges slowly there: energy within 0.5 %.
    assert abs(np.sum(s_rand ** 2) / np.sum(s_exact ** 2) - 1) < 5e-3
    np.testing.assert_allclose(a.T @ a, np.eye(16), atol=1e-10)   # orthonormal basis
    # with a spectral gap after k the randomized values are exact to rounding
    q1, _ = np.linalg.qr(rng.standard_normal((300, 16)))
    q2, _ = np.linalg.qr(rng.standard_normal((200, 16)))
    low = q1 @ np.diag(np.geomspace(100, 10, 16)) @ q2.T + 1e-3 * rng.standard_normal((300, 200))
    s_exact, _, _ = O.svd_topk(low, 16, method="exact")
    s_rand, _, _ = O.svd_topk(low, 16, method="randomized", seed=2)
    np.testing.assert_allclose(s_rand, s_exact, rtol=1e-9)


def test_perron_vector_one_signed():
    """P8 (Perron-Frobenius): the top singular pair of |R| (entrywise positive) is
    one-signed; with the sign convention it is non-negative."""
    rng = np.random.default_rng(2)
    mag = np.abs(rng.standard_normal((64, 48)))
    _, a, b = O.svd_topk(mag, 4)
    assert np.all(a[:, 0] > 0) and np.all(b[:, 0] > 0)


# ---------------------------------------------------------------- storage dtype
def test_bf16_rounding_nearest_even():
    """Reading R7: bf16 storage with round-to-nearest-even (ties to even)."""
    one = 1.0
    vals = np.array([one + 2 ** -8, one + 3 * 2 ** -8, one + 2 ** -8 + 2 ** -20, -2.5, 0.0])
    got = O.round_to_dtype(vals, "bf16")
    np.testing.assert_array_equal(got, [1.0, 1.0 + 4 * 2 ** -8, 1.0 + 2 ** -7, -2.5, 0.0])


def test_bf16_rounding_matches_torch():
    """Independent implementation: torch's float32 -> bfloat16 conversion (RNE)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(4096) * 10.0 ** rng.integers(-6, 6, 4096)).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(O.bf16_bits(x), want)


# ---------------------------------------------------------------- sign split / pack
def test_sign_split_zero_is_plus_one():
    """Eq.5: W = W_sign (.) |W|; SPEC S:187 example (reading R6)."""
    s, mag = O.sign_split(np.array([[-2.0, 0.0], [3.0, -1.0]]))
    np.testing.assert_array_equal(s, [[-1, 1], [1, -1]])
    np.testing.assert_array_equal(mag, [[2.0, 0.0], [3.0, 1.0]])


def test_pack_examples():
    """SPEC S:196-202."""
    np.testing.assert_array_equal(O.pack_signs(np.ones((2, 2), np.int8)), [0x0F])
    np.testing.assert_array_equal(O.pack_signs(np.array([[1, -1, 1]], np.int8)), [0x05])
    np.testing.assert_array_equal(O.unpack_signs(np.array([0x00], np.uint8), 2, 2), -np.ones((2, 2)))


def test_pack_brute_force_bit_order():
    """Canonical order (reading R11): bit j*d_in + c, LSB-first; pure-Python loop."""
    rng = np.random.default_rng(9)
    d_out, d_in = 5, 7
    s = np.where(rng.random((d_out, d_in)) < 0.5, -1, 1).astype(np.int8)
    want = [0] * ((d_out * d_in + 7) // 8)
    for j in range(d_out):
        for c in range(d_in):
            i = j * d_in + c
            if s[j, c] == 1:
                want[i // 8] |= 1 << (i % 8)
    np.testing.assert_array_equal(O.pack_signs(s), want)


def test_pack_round_trip_and_malformed():
    """SPEC S:198."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        d_out, d_in = rng.integers(1, 20, 2)
        s = np.where(rng.random((d_out, d_in)) < 0.5, -1, 1).astype(np.int8)
        np.testing.assert_array_equal(O.unpack_signs(O.pack_signs(s), d_out, d_in), s)
    with pytest.raises(O.MalformedBuffer):
        O.unpack_signs(np.array([0xFF], np.uint8), 1, 3)      # pad bits set
    with pytest.raises(O.MalformedBuffer):
        O.unpack_signs(np.array([0x01, 0x00], np.uint8), 1, 3)  # wrong length


# ---------------------------------------------------------------- Eq.5-8
def test_avd_rank1_exact_and_zero():
    """SPEC S:261-262 / P5: |R| rank-1 is restored exactly by one k=1 block;
    R = 0 gives zero factors and zero residual."""
    rng = np.random.default_rng(4)
    a = rng.uniform(0.5, 2.0, 12)
    b = rng.uniform(0.5, 2.0, 9)
    sg = np.where(rng.random((12, 9)) < 0.5, -1.0, 1.0)
    r = sg * np.outer(a, b)
    blk, r_next = O.avd_step(r, 1, dtype="f64")
    assert np.linalg.norm(r_next) < 1e-12 * np.linalg.norm(r)
    blk, r_next = O.avd_step(r, 1, dtype="bf16")
    assert np.linalg.norm(r_next) < 1e-2 * np.linalg.norm(r)
    blk0, r0 = O.avd_step(np.zeros((4, 5)), 2, dtype="f64")
    assert not np.any(blk0.u) and not np.any(blk0.v) and not np.any(r0)


def test_energy_identity_closed_form():
    """P2 (Eq.5-7 + Eckart-Young): since |S| = 1,
    ||R - S(.)(U V^T)||_F = || |R| - U V^T ||_F, so with unrounded factors
    ||R_i||^2 = ||R_{i-1}||^2 - sum_{r<=k} sigma_r(|R_{i-1}|)^2 exactly.
    A wrong sign, a missing sqrt(sigma) split or a transposed factor breaks it."""
    rng = np.random.default_rng(12)
    w = rng.standard_normal((40, 30))
    blocks = O.iavd(w, 6, 4, dtype="f64")
    prev = np.linalg.norm(w) ** 2
    for blk in blocks:
        after = blk.residual_norm_after ** 2
        assert after == pytest.approx(prev - np.sum(blk.sigma ** 2), rel=1e-9, abs=1e-9)
        prev = after


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16", "f16"])
@pytest.mark.parametrize("k", [1, 4, 16])
def test_residual_monotone(dtype, k):
    """P3 / SPEC S:284: ||W - W_hat_t||_F non-increasing in t (1e-3 slack)."""
    for seed in range(4):
        rng = np.random.default_rng(seed)
        m, n = rng.integers(17, 48, 2)
        w = rng.standard_normal((m, n))
        blocks = O.iavd(w, 16, min(k, m, n), dtype=dtype)
        prev = np.linalg.norm(w)
        for t in range(1, 17):
            err = np.linalg.norm(w - O.reconstruct(blocks, np.ones(n), t, m, n))
            assert err <= prev * (1 + 1e-3) + 1e-12
            prev = err


def test_full_rank_single_block_exact_and_eq4_end_to_end():
    """P4 (north star): k = min(d_out, d_in) makes one block exact; and through
    Eq.4 the oracle's y equals x W^T of the ORIGINAL (unscaled) W -- pins that
    1/s is applied to input channels at inference."""
    rng = np.random.default_rng(8)
    w = rng.standard_normal((10, 14)) * 0.02
    g = channel_gains(14, 1)
    x_cal = make_calibration(64, g, 2)
    s, blocks = O.compress(w, x_cal, 1, 10, dtype="f64")
    w_hat = O.reconstruct(blocks, s, 1, 10, 14)
    np.testing.assert_allclose(w_hat, w, rtol=0, atol=1e-13)
    x = make_x(3, g, 5)
    np.testing.assert_allclose(O.matmul_dense(blocks, s, 1, x), x @ w.T, rtol=1e-10, atol=1e-13)


def test_dense_equals_factored_equals_brute_force():
    """P6: dense W_hat x == factored sum_i sum_r u (.) S(v (.) x/s) == a pure-Python
    triple loop over (i, j, c, r) on a tiny case."""
    rng = np.random.default_rng(21)
    d_out, d_in, n, k, bsz = 6, 10, 3, 2, 2
    w = rng.standard_normal((d_out, d_in))
    x_cal = rng.standard_normal((20, d_in))
    s, blocks = O.compress(w, x_cal, n, k, dtype="bf16")
    x = rng.standard_normal((bsz, d_in))
    y_dense = O.matmul_dense(blocks, s, n, x)
    y_fact = O.matmul_factored(blocks, s, n, x)
    np.testing.assert_allclose(y_fact, y_dense, rtol=1e-12, atol=1e-14)
    y_bf = np.zeros((bsz, d_out))
    for b in range(bsz):
        for blk in blocks:
            sm = O.unpack_signs(blk.signs, d_out, d_in)
            for j in range(d_out):
                for c in range(d_in):
                    uv = sum(blk.u[j, r] * blk.v[c, r] for r in range(k))
                    y_bf[b, j] += sm[j, c] * uv * x[b, c] / s[c]
    np.testing.assert_allclose(y_dense, y_bf, rtol=1e-12, atol=1e-14)


def test_reconstruct_levels():
    """SPEC S:279-281 (P11): level 0 is zero; level t - level t-1 == block t;
    LevelOutOfRange outside [0, n]."""
    rng = np.random.default_rng(6)
    w = rng.standard_normal((8, 12))
    blocks = O.iavd(w, 4, 3, dtype="bf16")
    ones = np.ones(12)
    assert not np.any(O.reconstruct(blocks, ones, 0, 8, 12))
    for t in range(1, 5):
        diff = O.reconstruct(blocks, ones, t, 8, 12) - O.reconstruct(blocks, ones, t - 1, 8, 12)
        np.testing.assert_allclose(diff, O.restore_block(blocks[t - 1], 8, 12), atol=1e-12)
    with pytest.raises(O.LevelOutOfRange):
        O.reconstruct(blocks, ones, 5, 8, 12)


def test_incremental_walk_equals_fresh():
    """P12 / SPEC S:418: a random load/offload walk (add or subtract restored
    blocks, offload in reverse order) ends equal to fresh reconstruction."""
    rng = np.random.default_rng(13)
    w = rng.standard_normal((9, 11))
    blocks = O.iavd(w, 8, 2, dtype="f32")
    ones = np.ones(11)
    cur, level = np.zeros((9, 11)), 0
    for _ in range(50):
        target = int(rng.integers(0, 9))
        while level < target:
            cur += O.restore_block(blocks[level], 9, 11)
            level += 1
        while level > target:
            level -= 1
            cur -= O.restore_block(blocks[level], 9, 11)
        np.testing.assert_allclose(cur, O.reconstruct(blocks, ones, level, 9, 11), atol=1e-9)


def test_avd_beats_size_matched_svd():
    """P13 (Fig.5 ablation): one AVD block (k=16) beats vanilla
    SVD with k' = k + ceil(mn / (16 (m+n))) in >= 90 of 100 random 64x64 cases."""
    wins = 0
    for seed in range(100):
        w = np.random.default_rng(seed).standard_normal((64, 64))
        kp = 16 + int(np.ceil(64 * 64 / (16 * 128)))
        blk, r = O.avd_step(w, 16, dtype="f16")
        A, B, _ = O.rank_k_factors(w, kp)
        svd_err = np.linalg.norm(w - O.round_to_dtype(A, "f16") @ O.round_to_dtype(B, "f16").T)
        wins += np.linalg.norm(r) < svd_err
    assert wins >= 90


def test_c1_brute_force_exact_loop():
    """P14: config C1 (256x512, n=4, k=16, fp32 factors) with exact LAPACK SVD:
    every sign is +-1, pad bits are zero, residual decreases, dense == factored."""
    g = channel_gains(512, 1004)
    w = make_weight(256, 512, 1000)
    x_cal = make_calibration(512, g, 1001)
    s, blocks = O.compress(w, x_cal, 4, 16, dtype="f32")
    norms = [blocks[0].residual_norm_before] + [b.residual_norm_after for b in blocks]
    assert all(a > b for a, b in zip(norms, norms[1:]))
    for blk in blocks:
        assert blk.signs.size == 256 * 512 // 8
        sm = O.unpack_signs(blk.signs, 256, 512)
        assert set(np.unique(sm)) <= {-1, 1}
    x = make_x(1, g, 1002)
    np.testing.assert_allclose(O.matmul_factored(blocks, s, 4, x), O.matmul_dense(blocks, s, 4, x),
                               rtol=1e-11)


def test_relative_l2_metric():
    """Reading R16: per-row relative L2, max over rows; zero reference -> exact."""
    assert O.relative_l2([[3.0, 4.0]], [[3.0, 4.0]]) == 0.0
    assert O.relative_l2([[3.0, 4.0], [1, 0]], [[3.0, 4.0], [2, 0]]) == pytest.approx(0.5)
    assert O.relative_l2([[0.0, 0.0]], [[0.0, 0.0]]) == 0.0
    assert O.relative_l2([[1e-30, 0.0]], [[0.0, 0.0]]) == float("inf")
    assert O.relative_l2([[np.nan, 1.0]], [[1.0, 1.0]]) == float("inf")   # NaN never passes
    assert O.relative_l2([[1.0, 1.0]], [[np.inf, 1.0]]) == float("inf")
    with pytest.raises(ValueError):
        O.relative_l2([[1.0, 2.0]], [[1.0, 2.0, 3.0]])
