"""Seeded shape / level / batch / dtype fuzzing of bitstack_matmul against the CPU oracle.

Random stored-form blocks (synthetic.make_random_blocks, the bench's generator) on random
shapes -- ragged d_out, ragged d_in (multiples of 8 take the tensor-core paths, others the
SIMT path), k in {1, 4, 8, 16, 20, 32}, factor dtypes bf16 / f16 / f32, levels 0..n, batches
1..20 (decode, chunked decode and prefill), row shards -- all checked against the oracle's
dense definition (Eq.8 + Eq.4) at the bar of the factor dtype.
"""
import numpy as np
import pytest

from bitstack_test_helpers import blocks_from_arrays
from oracle import bitstack_oracle as O
from synthetic import make_random_blocks

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_23918_b200 import build
    build.build()
    import paper_2410_23918_b200 as pkg
    pkg.load_library()
    return pkg


def _stored(dtype, u, v):
    if dtype == "bf16":
        return O.bf16_bits(u), O.bf16_bits(v), O.round_to_dtype(u, "bf16"), O.round_to_dtype(v, "bf16")
    if dtype == "f16":
        return u.astype(np.float16), v.astype(np.float16), O.round_to_dtype(u, "f16"), O.round_to_dtype(v, "f16")
    return u.astype(np.float32), v.astype(np.float32), u.astype(np.float32).astype(np.float64), \
        v.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("case", range(64))
def test_fuzz(bs, case):
    rng = np.random.default_rng(7000 + case)
    d_out = int(rng.integers(1, 700))
    d_in = int(rng.choice([8 * int(rng.integers(1, 160)), int(rng.integers(1, 900))]))
    k = int(min(rng.choice([1, 4, 8, 16, 16, 20, 32]), d_out, d_in))
    dtype = str(rng.choice(["bf16", "bf16", "f16", "f32"]))
    n = int(rng.integers(1, 6))
    signs, u, v, s = make_random_blocks(n, d_out, d_in, k, seed=8000 + case)
    us, vs, ur, vr = _stored(dtype, u, v)
    blocks = blocks_from_arrays(signs, ur, vr)
    r0 = int(rng.integers(0, d_out))
    r1 = int(rng.integers(r0 + 1, d_out + 1)) if rng.random() < 0.4 else d_out
    r0 = r0 if r1 != d_out or rng.random() < 0.3 else 0
    lay = bs.Layer(d_out, d_in, k=k, n_capacity=n, factor_dtype=dtype, row_begin=r0, row_end=r1)
    lay.load_blocks(0, signs, torch.from_numpy(np.ascontiguousarray(us).view(np.int16)) if dtype == "bf16" else us,
                    torch.from_numpy(np.ascontiguousarray(vs).view(np.int16)) if dtype == "bf16" else vs, s)
    s64 = s.astype(np.float64)
    tol = 1e-5 if dtype == "f32" else 1e-3
    for _ in range(3):
        level = int(rng.integers(0, n + 1))
        batch = int(rng.choice([1, 2, 3, 4, 5, 9, 17, 20]))
        lay.set_num_blocks(level)
        x = torch.from_numpy(rng.standard_normal((batch, d_in)).astype(np.float32)).cuda()
        y = lay.matmul(x)
        torch.cuda.synchronize()
        yn = y.cpu().numpy().astype(np.float64)
        if level == 0:
            assert not np.any(yn)
            continue
        ref = O.matmul_dense(blocks, s64, level, x.cpu().numpy().astype(np.float64))[:, r0:r1]
        err = O.relative_l2(yn, ref)
        assert err <= tol, (d_out, d_in, k, dtype, n, level, batch, (r0, r1), err)
    lay.close()
