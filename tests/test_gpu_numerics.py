"""GPU numerics under dynamic range: bitstack_matmul against the CPU oracle when x, s and the
batch span many binades (VERDICT r1 "next round" item 1).

The oracle is scale-equivariant (Eq.4: y = W_s (x / s)), so every case below has
the same relative-L2 bar as the ordinary parity tests (reading R16): 1e-3 with bf16 / f16
factors, 1e-5 with fp32 factors, y in fp32.  Paths: the MX e4m3 decode (per-(K-block, column,
digit) scales), the fp16 decode of fp32-factor layers and the prefill GEMM (power-of-two
operand scales from the call's max |x / s|), the restore-and-multiply kernel (tf32 operands, fp32
range), and the SIMT kernel (fp32 throughout).

Also the bit-exact pin of the decode kernel's sign expansion ("unpacked ... for
use during inference"): with U_i[:, 0] = 2^i, V_i[:, 0] = 1, s = 1 and a one-hot x = e_c,
bitstack_matmul returns sum_i 2^i S_i[:, c] exactly, which decodes to every sign bit.
"""
import numpy as np
import pytest

from bitstack_test_helpers import stack_blocks
from oracle import bitstack_oracle as O
from synthetic import channel_gains, make_calibration, make_weight, make_x, random_signs_bytes

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


_CASES = {}


def case(d_out, d_in, n, dtype, seed, k=16):
    key = (d_out, d_in, n, dtype, seed, k)
    if key not in _CASES:
        g = channel_gains(d_in, seed + 4)
        w = make_weight(d_out, d_in, seed)
        x_cal = make_calibration(max(256, d_in), g, seed + 1)
        s, blocks = O.compress(w, x_cal, n, k, dtype=dtype, method="exact", seed=seed)
        _CASES[key] = (g, s.astype(np.float32), blocks)
    return _CASES[key]


def layer(bs, d_out, d_in, blocks, s32, dtype, kernel="auto"):
    signs, u, v = stack_blocks(blocks, dtype)
    lay = bs.Layer(d_out, d_in, k=int(u.shape[-1]), n_capacity=len(blocks), factor_dtype=dtype)
    lay.load_blocks(0, signs, u, v, s32)
    if kernel != "auto":
        lay.set_kernel(kernel)
    torch.cuda.synchronize()
    return lay


def run(lay, x64, x_dtype=torch.float32):
    x = torch.from_numpy(np.ascontiguousarray(x64, dtype=np.float32)).to(x_dtype).cuda()
    y = lay.matmul(x)
    torch.cuda.synchronize()
    return y.double().cpu().numpy(), x.double().cpu().numpy()


def check(lay, blocks, s32, n, x64, tol, x_dtype=torch.float32):
    y, xr = run(lay, x64, x_dtype)
    ref = O.matmul_dense(blocks, s32.astype(np.float64), n, xr)
    err = O.relative_l2(y, ref)
    assert err <= tol, err
    return err


TOL = {"bf16": 1e-3, "f16": 1e-3, "f32": 1e-5}
# (path name, factor dtype, kernel): the MX e4m3 decode, the fp16 decode (fp32 factors), the
# prefill GEMM (forced at small batches), the SIMT kernel
PATHS = [("mx", "bf16", "tc"), ("mx16", "f16", "tc"), ("fp16dec", "f32", "tc"), ("prefill", "bf16", "prefill"),
         ("prefill16", "f16", "prefill"), ("rgemv", "bf16", "rgemv"), ("rgemv16", "f16", "rgemv"), ("simt", "bf16", "simt")]


@pytest.mark.parametrize("path,dtype,kernel", PATHS)
@pytest.mark.parametrize("j", [-40, -20, 0, 20, 40])
def test_x_scale_sweep(bs, path, dtype, kernel, j):
    """x 2^j for j in -40..40: y scales exactly, the error bar does not move."""
    g, s32, blocks = case(384, 640, 4, dtype, 9001)
    lay = layer(bs, 384, 640, blocks, s32, dtype, kernel)
    x = make_x(3, g, 5) * 2.0 ** j
    check(lay, blocks, s32, 4, x, TOL[dtype])


@pytest.mark.parametrize("path,dtype,kernel", PATHS)
@pytest.mark.parametrize("e", [-10, 10])
def test_s_scale_sweep(bs, path, dtype, kernel, e):
    """s 2^e: W_hat = W_s diag(1/s) shrinks / grows by 2^-e (Eq.4); y follows exactly."""
    g, s32, blocks = case(384, 640, 4, dtype, 9002)
    s2 = (s32 * np.float32(2.0 ** e)).astype(np.float32)
    lay = layer(bs, 384, 640, blocks, s2, dtype, kernel)
    check(lay, blocks, s2, 4, make_x(2, g, 6), TOL[dtype])


@pytest.mark.parametrize("path,dtype,kernel", PATHS)
@pytest.mark.parametrize("pattern", ["chunk_up", "chunk_down", "one_hot", "outlier"])
def test_dynamic_range_within_a_token(bs, path, dtype, kernel, pattern):
    """One token whose channels span 2^24: a 128-column chunk x 2^12, a chunk x 2^-12, a single
    non-zero entry, or one channel 2^12 above the rest."""
    g, s32, blocks = case(512, 1024, 5, dtype, 9003)
    lay = layer(bs, 512, 1024, blocks, s32, dtype, kernel)
    x = make_x(2, g, 7)
    if pattern == "chunk_up":
        x[:, 256:384] *= 2.0 ** 12
    elif pattern == "chunk_down":
        x[:, 512:640] *= 2.0 ** -12
    elif pattern == "one_hot":
        x[:] = 0.0
        x[0, 777] = 3.0
        x[1, 5] = -2.0 ** -20
    else:
        x[:, 901] *= 2.0 ** 12
    check(lay, blocks, s32, 5, x, TOL[dtype])


@pytest.mark.parametrize("path,dtype,kernel", PATHS)
@pytest.mark.parametrize("batch", [2, 3, 4, 8])
def test_tokens_far_apart_in_one_batch(bs, path, dtype, kernel, batch):
    """Tokens 2^12 apart in one call: each token keeps its own bar (per-token error)."""
    g, s32, blocks = case(384, 640, 3, dtype, 9004)
    lay = layer(bs, 384, 640, blocks, s32, dtype, kernel)
    x = make_x(batch, g, 8)
    for b in range(batch):
        x[b] *= 2.0 ** (12 * (b % 3) - 12)
    check(lay, blocks, s32, 3, x, TOL[dtype])


def test_grouped_and_k32_dynamic_range(bs):
    """Grouped launches and k = 32 (fused rank halves at batch 1) under the same x patterns."""
    cases = [case(512, 640, 3, "bf16", 9005), case(300, 640, 2, "bf16", 9006)]
    lays = [layer(bs, 512, 640, cases[0][2], cases[0][1], "bf16"),
            layer(bs, 300, 640, cases[1][2], cases[1][1], "bf16")]
    for batch in (1, 3):
        x = make_x(batch, cases[0][0], 9)
        x[:, 128:256] *= 2.0 ** 12
        x[-1] *= 2.0 ** -12
        xs = [torch.from_numpy(x.astype(np.float32)).cuda()] * 2
        ys = bs.matmul_grouped(lays, xs)
        torch.cuda.synchronize()
        for (g, s32, blocks), lay, y in zip(cases, lays, ys):
            ref = O.matmul_dense(blocks, s32.astype(np.float64), lay.info()["n_active"], x.astype(np.float32).astype(np.float64))
            assert O.relative_l2(y.double().cpu().numpy(), ref) <= 1e-3
    g, s32, blocks = case(256, 512, 3, "bf16", 9007, k=32)
    lay = layer(bs, 256, 512, blocks, s32, "bf16")
    for batch in (1, 2):
        x = make_x(batch, g, 10)
        x[:, 0:128] *= 2.0 ** 12
        check(lay, blocks, s32, 3, x, 1e-3)


# ------------------------------------------------------------------ bit-exact decode pin
@pytest.mark.parametrize("k,factor_dtype", [(16, "bf16"), (16, "f16"), (32, "bf16"), (16, "f32")])
def test_decode_sign_expansion_bit_exact(bs, k, factor_dtype):
    """U_i[:,0] = 2^i, V_i[:,0] = 1 (other ranks 0), s = 1, x = e_c: y = sum_i 2^i S_i[:, c],
    integers below 2^16, exact through the decode kernels (MX e4m3 for bf16 / f16 factors, with
    the fused N = 96 geometry for k = 32 at batch 1; fp16 for fp32 factors).  Decoding y gives
    back every canonical bit of every block."""
    d_out, d_in, n = 256, 384, 14
    signs = random_signs_bytes(n, d_out, d_in, seed=77 + k)
    u = np.zeros((n, d_out, k), np.float32)
    v = np.zeros((n, d_in, k), np.float32)
    for i in range(n):
        u[i, :, 0] = 2.0 ** i
        v[i, :, 0] = 1.0
    lay = bs.Layer(d_out, d_in, k=k, n_capacity=n, factor_dtype=factor_dtype)
    if factor_dtype == "bf16":
        uu, vv = O.bf16_bits(u), O.bf16_bits(v)
    elif factor_dtype == "f16":
        uu, vv = u.astype(np.float16), v.astype(np.float16)
    else:
        uu, vv = u, v
    lay.load_blocks(0, signs, uu, vv, np.ones(d_in, np.float32))
    lay.set_kernel("tc")
    want = [np.unpackbits(signs[i], bitorder="little")[: d_out * d_in].reshape(d_out, d_in) for i in range(n)]
    cols = range(d_in) if k == 16 else range(0, d_in, 5)
    eye = np.eye(d_in, dtype=np.float32)
    if k == 16:   # all one-hot tokens in batches of 8 (the widest decode batch)
        y, _ = run(lay, eye)
        ycols = y.T                         # [d_out, d_in]: column c = response to e_c
    else:         # batch 1 takes the fused two-half geometry
        ycols = np.zeros((d_out, d_in))
        for c in cols:
            ycols[:, c] = run(lay, eye[c:c + 1])[0][0]
    for c in cols:
        w = np.rint(ycols[:, c]).astype(np.int64)
        assert np.array_equal(w.astype(np.float64), ycols[:, c]), c      # exact integers
        code = (w + (2 ** n - 1)) // 2
        for i in range(n):
            np.testing.assert_array_equal((code >> i) & 1, want[i][:, c])


# ------------------------------------------------------------------ one handle, several streams
def test_calls_on_one_handle_from_two_streams(bs):
    """A handle's workspaces are reused by every call; calls issued on alternating streams must be
    ordered by the library (include/bitstack.h conventions) and give the single-stream results."""
    g, s32, blocks = case(512, 1024, 4, "bf16", 9100)
    lay = layer(bs, 512, 1024, blocks, s32, "bf16")
    xs = [torch.from_numpy(make_x(b, g, 200 + i).astype(np.float32)).cuda() for i, b in enumerate([1, 3, 1, 8, 2, 20] * 3)]
    ref = []
    for x in xs:
        ref.append(lay.matmul(x).clone())
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for i, x in enumerate(xs):
        st = s1 if i % 2 == 0 else s2
        y = torch.empty((x.shape[0], 512), dtype=torch.float32, device="cuda")
        y.record_stream(st)
        lay.matmul_raw(x.data_ptr(), bs.F32, y.data_ptr(), bs.F32, x.shape[0], st.cuda_stream)
        outs.append(y)
    torch.cuda.synchronize()
    for y, r in zip(outs, ref):
        assert torch.equal(y, r)
