"""GPU parity: bitstack_matmul / bitstack_reconstruct (CUDA, through the C ABI)
against the CPU oracle on the SAME stored blocks and the SAME x.

Tolerances (north star): relative L2 per batch row (reading R16)
  <= 1e-3 with bf16/f16 factors, <= 1e-5 with fp32 factors, y in fp32;
  bf16 y adds its own rounding (1.7e-3 measured on the oracle) -> 4e-3.
Sign unpacking is checked bit-exactly (P15), with no float tolerance.
"""
import os
import numpy as np
import pytest

from bitstack_test_helpers import blocks_from_arrays, stack_blocks
from oracle import bitstack_oracle as O
from synthetic import (channel_gains, make_calibration, make_random_blocks, make_weight, make_x,
                       random_signs_bytes, seed_for)

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


def compress_case(d_out, d_in, n, dtype, seed, method="exact", p=None, k=16):
    g = channel_gains(d_in, seed + 4)
    w = make_weight(d_out, d_in, seed)
    x_cal = make_calibration(p or max(256, d_in), g, seed + 1)
    s, blocks = O.compress(w, x_cal, n, k, dtype=dtype, method=method, seed=seed)
    s32 = s.astype(np.float32)
    return g, s32, blocks


def make_layer(bs, d_out, d_in, blocks, s32, dtype, n_capacity=None, row_begin=0, row_end=None):
    signs, u, v = stack_blocks(blocks, dtype)
    lay = bs.Layer(d_out, d_in, k=int(u.shape[-1]), n_capacity=n_capacity or len(blocks), factor_dtype=dtype,
                   row_begin=row_begin, row_end=row_end)
    lay.load_blocks(0, signs, u, v, s32)
    torch.cuda.synchronize()
    return lay


def oracle_y(blocks, s32, n, x):
    return O.matmul_dense(blocks, s32.astype(np.float64), n, x)


def gpu_y(lay, x_np, x_dtype=torch.float32, y_dtype=torch.float32):
    x = torch.from_numpy(np.ascontiguousarray(x_np, dtype=np.float32)).to(x_dtype).cuda()
    y = lay.matmul(x, y_dtype=y_dtype)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64), x.float().cpu().numpy().astype(np.float64)


# ------------------------------------------------------------------ P15: bit-exact unpack
@pytest.mark.parametrize("factor_dtype", ["f32", "bf16"])   # device sign layouts F16 and F8
@pytest.mark.parametrize("shape", [(256, 384), (300, 200), (128, 1000)])
def test_sign_unpack_bit_exact(bs, shape, factor_dtype):
    """U_i[:,0] = 2^i, V_i[:,0] = 1, other columns 0, s = 1  =>  reconstruct in fp32
    gives sum_i 2^i S_i exactly; decoding it must give back every canonical bit."""
    d_out, d_in = shape
    n = 16
    signs = random_signs_bytes(n, d_out, d_in, seed=7 + d_out)
    u = np.zeros((n, d_out, 16), np.float32)
    v = np.zeros((n, d_in, 16), np.float32)
    for i in range(n):
        u[i, :, 0] = 2.0 ** i
        v[i, :, 0] = 1.0
    lay = bs.Layer(d_out, d_in, k=16, n_capacity=n, factor_dtype=factor_dtype)
    if factor_dtype == "bf16":
        u, v = O.bf16_bits(u), O.bf16_bits(v)   # powers of two: exact in bf16
    lay.load_blocks(0, signs, u, v, np.ones(d_in, np.float32))
    w = lay.reconstruct(torch.float32).cpu().numpy().astype(np.int64)
    # decode: w = sum_i 2^i (2 b_i - 1) = 2 sum_i 2^i b_i - (2^n - 1)
    code = (w + (2 ** n - 1)) // 2
    assert np.all((w + (2 ** n - 1)) % 2 == 0)
    for i in range(n):
        bits = (code >> i) & 1
        want = np.unpackbits(signs[i], bitorder="little")[: d_out * d_in].reshape(d_out, d_in)
        np.testing.assert_array_equal(bits, want)


# ------------------------------------------------------------------ C1: fp32 factors, 1e-5
@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_c1_parity_fp32(bs, kernel):
    """Config C1 (256x512, n=4, k=16, fp32 factors, exact LAPACK loop), batch 1."""
    g, s32, blocks = compress_case(256, 512, 4, "f32", seed_for(1))
    lay = make_layer(bs, 256, 512, blocks, s32, "f32")
    lay.set_kernel(kernel)
    x = make_x(1, g, seed_for(1, 0, "x"))
    for n in range(0, 5):
        lay.set_num_blocks(n)
        y, xr = gpu_y(lay, x)
        ref = oracle_y(blocks, s32, n, xr)
        if n == 0:
            assert not np.any(y)
        else:
            assert O.relative_l2(y, ref) <= 1e-5, (n, O.relative_l2(y, ref))


# ------------------------------------------------------------------ ragged shapes, batches
@pytest.mark.parametrize("shape", [(384, 640), (200, 296), (1100, 264)])
@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_bf16_parity_ragged(bs, shape, kernel):
    d_out, d_in = shape
    g, s32, blocks = compress_case(d_out, d_in, 5, "bf16", 31 + d_out)
    lay = make_layer(bs, d_out, d_in, blocks, s32, "bf16")
    lay.set_kernel(kernel)
    for batch in (1, 2, 3, 5, 8, 16, 17):
        x = make_x(batch, g, 77 + batch)
        y, xr = gpu_y(lay, x)
        ref = oracle_y(blocks, s32, 5, xr)
        assert O.relative_l2(y, ref) <= 1e-3, (batch, O.relative_l2(y, ref))


def test_unaligned_d_in_uses_simt(bs):
    """d_in % 8 != 0: the TMA-fed tcgen05 path is refused (E_UNSUPPORTED when forced) and
    AUTO runs the SIMT kernel -- still within tolerance."""
    g, s32, blocks = compress_case(200, 300, 3, "bf16", 44)
    lay = make_layer(bs, 200, 300, blocks, s32, "bf16")
    x = make_x(2, g, 1)
    y, xr = gpu_y(lay, x)
    assert O.relative_l2(y, oracle_y(blocks, s32, 3, xr)) <= 1e-3
    lay.set_kernel("tc")
    with pytest.raises(bs.BitStackError) as e:
        gpu_y(lay, x)
    assert e.value.name == "E_UNSUPPORTED"


@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_fp32_factor_batches(bs, kernel):
    """fp32 factors use two fp16 digits of Z on the tensor-core path: 1e-5 at every batch."""
    g, s32, blocks = compress_case(384, 512, 3, "f32", 91)
    lay = make_layer(bs, 384, 512, blocks, s32, "f32")
    lay.set_kernel(kernel)
    for batch in (1, 2, 4, 7, 8, 9):
        x = make_x(batch, g, 5 + batch)
        y, xr = gpu_y(lay, x)
        assert O.relative_l2(y, oracle_y(blocks, s32, 3, xr)) <= 1e-5


def test_f16_factors_and_dtypes(bs):
    """Paper's own FP16 factors; bf16/f16 activations; bf16 output."""
    g, s32, blocks = compress_case(256, 384, 4, "f16", 55)
    lay = make_layer(bs, 256, 384, blocks, s32, "f16")
    x = make_x(3, g, 8)
    for xdt in (torch.float32, torch.bfloat16, torch.float16):
        y, xr = gpu_y(lay, x, x_dtype=xdt)
        assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 1e-3
    y, xr = gpu_y(lay, x, y_dtype=torch.bfloat16)
    assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 4e-3


# ------------------------------------------------------------------ C2: every n, full size
@pytest.fixture(scope="module")
def c2(bs):
    g, s32, blocks = compress_case(4096, 4096, 16, "bf16", seed_for(2), method="randomized", p=4096)
    lay = make_layer(bs, 4096, 4096, blocks, s32, "bf16")
    return g, s32, blocks, lay


def test_c2_parity_every_n(c2):
    """Config C2 (Llama-3.1-8B q_proj 4096x4096, n=1..16, B=1): <= 1e-3 at every n,
    in the launch configuration bench.py times (auto kernel = tcgen05)."""
    g, s32, blocks, lay = c2
    x = make_x(1, g, seed_for(2, 0, "x"))
    xt = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).cuda()
    xr = xt.float().cpu().numpy().astype(np.float64)
    partial = [O.matmul_dense([b], s32.astype(np.float64), 1, xr) for b in blocks]  # Eq.8 is a sum
    ref = np.zeros_like(partial[0])
    for n in range(1, 17):
        ref = ref + partial[n - 1]
        lay.set_num_blocks(n)
        y = lay.matmul(xt).cpu().numpy().astype(np.float64)
        err = O.relative_l2(y, ref)
        assert err <= 1e-3, (n, err)


def test_c2_reconstruct_matches_oracle(c2):
    g, s32, blocks, lay = c2
    lay.set_num_blocks(3)
    w = lay.reconstruct(torch.float32).cpu().numpy().astype(np.float64)
    ref = O.reconstruct(blocks, s32.astype(np.float64), 3, 4096, 4096)
    assert np.linalg.norm(w - ref) / np.linalg.norm(ref) <= 1e-6


# ------------------------------------------------------------------ stack semantics
def test_incremental_load_offload_walk(bs):
    """Blocks pushed one at a time, random set_num_blocks walk, re-push after offload:
    y always equals the oracle at the active level."""
    g, s32, blocks = compress_case(256, 256, 6, "bf16", 123)
    signs, u, v = stack_blocks(blocks, "bf16")
    lay = bs.Layer(256, 256, k=16, n_capacity=6, factor_dtype="bf16")
    x = make_x(2, g, 4)
    rng = np.random.default_rng(0)
    lay.load_blocks(0, signs[:1], u[:1], v[:1], s32)
    resident = 1
    for step in range(30):
        if resident < 6 and rng.random() < 0.4:
            lay.load_blocks(resident, signs[resident:resident + 1], u[resident:resident + 1], v[resident:resident + 1])
            resident += 1
        n = int(rng.integers(0, resident + 1))
        lay.set_num_blocks(n)
        y, xr = gpu_y(lay, x)
        ref = oracle_y(blocks, s32, n, xr)
        if n == 0:
            assert not np.any(y)
        else:
            assert O.relative_l2(y, ref) <= 1e-3
    # offload to 2 then re-push block 2 (overwrites in place)
    lay.set_num_blocks(2)
    lay.load_blocks(2, signs[2:3], u[2:3], v[2:3])
    assert lay.info()["n_resident"] == 3
    lay.set_num_blocks(3)
    y, xr = gpu_y(lay, x)
    assert O.relative_l2(y, oracle_y(blocks, s32, 3, xr)) <= 1e-3


def test_errors_and_edge_cases(bs):
    g, s32, blocks = compress_case(128, 256, 3, "bf16", 9)
    signs, u, v = stack_blocks(blocks, "bf16")
    lay = bs.Layer(128, 256, k=16, n_capacity=3, factor_dtype="bf16")
    with pytest.raises(bs.BitStackError) as e:
        lay.set_num_blocks(1)
    assert e.value.name == "E_LEVEL_OUT_OF_RANGE"
    with pytest.raises(bs.BitStackError) as e:           # s required for block 0
        lay.load_blocks(0, signs, u, v, None)
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(bs.BitStackError) as e:           # first_block > resident
        lay.load_blocks(1, signs[:1], u[:1], v[:1])
    assert e.value.name == "E_LEVEL_OUT_OF_RANGE"
    lay.load_blocks(0, signs, u, v, s32)
    with pytest.raises(bs.BitStackError) as e:           # capacity
        lay.load_blocks(3, signs[:1], u[:1], v[:1])
    assert e.value.name == "E_CAPACITY"
    bad = np.zeros((1, (127 * 255 + 7) // 8), np.uint8)
    bad[0, -1] = 0xFF                                      # pad bits set
    lay2 = bs.Layer(127, 255, k=16, n_capacity=1, factor_dtype="bf16")
    with pytest.raises(bs.BitStackError) as e:
        lay2.load_blocks(0, bad, np.zeros((1, 127, 16), np.uint16), np.zeros((1, 255, 16), np.uint16),
                         np.ones(255, np.float32))
    assert e.value.name == "E_MALFORMED_BUFFER"
    s_bad = s32.copy()
    s_bad[3] = 0.0
    with pytest.raises(bs.BitStackError):
        lay.load_blocks(0, signs, u, v, s_bad)
    # batch 0 is a no-op, n = 0 gives exact zeros
    x = torch.zeros((0, 256), device="cuda")
    y = lay.matmul(x)
    assert y.shape == (0, 128)
    lay.set_num_blocks(0)
    y, _ = gpu_y(lay, make_x(4, g, 1))
    assert not np.any(y)


def test_row_shards_concatenate_to_full(bs):
    """Row sharding: shards [r0, r1) computed independently and
    concatenated equal the unsharded layer (no collective needed on one GPU)."""
    g, s32, blocks = compress_case(640, 384, 4, "bf16", 17)
    x = make_x(3, g, 2)
    full = make_layer(bs, 640, 384, blocks, s32, "bf16")
    yf, xr = gpu_y(full, x)
    cuts = [0, 128, 200, 512, 640]
    parts = []
    for a, b in zip(cuts, cuts[1:]):
        sh = make_layer(bs, 640, 384, blocks, s32, "bf16", row_begin=a, row_end=b)
        parts.append(gpu_y(sh, x)[0])
    ys = np.concatenate(parts, axis=1)
    ref = oracle_y(blocks, s32, 4, xr)
    assert O.relative_l2(ys, ref) <= 1e-3
    assert O.relative_l2(ys, yf) <= 1e-5


# ------------------------------------------------------------------ Zq edge cases
def test_zero_activation_segments(bs):
    """All-zero 128-column segments of x give all-zero Zq units (sentinel exponent): the
    decode kernel must skip them when choosing its scale reference and still match the
    oracle; an all-zero x gives y == 0 exactly."""
    g, s32, blocks = compress_case(512, 640, 4, "bf16", 91)
    lay = make_layer(bs, 512, 640, blocks, s32, "bf16")
    for batch in (1, 2, 4):
        x = make_x(batch, g, 11 + batch)
        x[:, :256] = 0.0            # first two subchunks empty: the CTAs' first units are sentinels
        x[:, 384:512] = 0.0
        y, xr = gpu_y(lay, x, x_dtype=torch.bfloat16)
        assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 1e-3, batch
    y, _ = gpu_y(lay, np.zeros((3, 640)), x_dtype=torch.bfloat16)
    assert not np.any(y)


# ------------------------------------------------------------------ host buffers (e2e path)
@pytest.mark.parametrize("batch", [1, 3, 12, 40])
def test_host_buffers(bs, batch):
    """bitstack_matmul with host x / y: pinned buffers (read / written in place by the decode and
    restore-and-multiply kernels, or staged for the prefill path) and pageable ones (staged) give
    the same y as device buffers."""
    g, s32, blocks = compress_case(256, 384, 3, "bf16", 81)
    lay = make_layer(bs, 256, 384, blocks, s32, "bf16")
    x = torch.from_numpy(make_x(batch, g, 5).astype(np.float32)).to(torch.bfloat16)
    y_dev = lay.matmul(x.cuda()).cpu()
    for pinned in (True, False):
        xh = x.pin_memory() if pinned else x.clone()
        yh = torch.empty((batch, 256), dtype=torch.float32)
        yh = yh.pin_memory() if pinned else yh
        lay.matmul_raw(xh.data_ptr(), bs.BF16, yh.data_ptr(), bs.F32, batch, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        np.testing.assert_allclose(yh.numpy(), y_dev.numpy(), rtol=1e-6, atol=1e-6)
    ref = oracle_y(blocks, s32, 3, x.float().numpy().astype(np.float64))
    assert O.relative_l2(y_dev.numpy().astype(np.float64), ref) <= 1e-3


# ------------------------------------------------------------------ block streaming (async load)
@pytest.mark.parametrize("shape,rows", [((640, 1024), None), ((520, 1000), (130, 390)), ((300, 200), (0, 300)),
                                        ((256, 100), (64, 256))])
def test_async_load_streaming_matches_sync(bs, shape, rows):
    """bitstack_load_blocks_async from pinned host memory on a side stream, blocks pushed in
    pieces (row shards with d_in % 8 == 0 copy only the shard's bytes; d_in % 8 != 0 falls
    back to full-block staging): after the stream passes, the device state is bit-identical
    to the synchronous load (fp32 reconstruct compared exactly) and y matches the oracle."""
    d_out, d_in = shape
    r0, r1 = rows or (0, d_out)
    g, s32, blocks = compress_case(d_out, d_in, 5, "bf16", 151 + d_in)
    signs, u, v = stack_blocks(blocks, "bf16")
    ref_lay = bs.Layer(d_out, d_in, k=16, n_capacity=5, factor_dtype="bf16", row_begin=r0, row_end=r1)
    ref_lay.load_blocks(0, signs, u, v, s32)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16) if a.dtype == np.uint16 else np.ascontiguousarray(a)).pin_memory()
    ps, pu, pv, pss = pin(signs), pin(u), pin(v), pin(s32)
    lay = bs.Layer(d_out, d_in, k=16, n_capacity=5, factor_dtype="bf16", row_begin=r0, row_end=r1)
    side = torch.cuda.Stream()
    lay.load_blocks_async(0, ps[:2], pu[:2], pv[:2], pss, stream=side)
    assert lay.info()["n_resident"] == 2
    lay.load_blocks_async(2, ps[2:], pu[2:], pv[2:], stream=side)
    ev = torch.cuda.Event()
    ev.record(side)
    torch.cuda.current_stream().wait_event(ev)
    assert lay.info()["n_resident"] == 5
    for n in (1, 3, 5):
        lay.set_num_blocks(n)
        ref_lay.set_num_blocks(n)
        assert torch.equal(lay.reconstruct(torch.float32), ref_lay.reconstruct(torch.float32))
    x = make_x(2, g, 8)
    y, xr = gpu_y(lay, x)
    full = oracle_y(blocks, s32, 5, xr)
    assert O.relative_l2(y, full[:, r0:r1]) <= 1e-3


def test_async_load_overlaps_matmul_on_another_stream(bs):
    """Streaming a new block into one handle on a side stream while another handle keeps
    computing on the main stream; the new level is used only after an event wait."""
    g, s32, blocks = compress_case(512, 1024, 4, "bf16", 171)
    signs, u, v = stack_blocks(blocks, "bf16")
    busy = make_layer(bs, 512, 1024, blocks, s32, "bf16")
    lay = make_layer(bs, 512, 1024, blocks[:2], s32, "bf16", n_capacity=4)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16) if a.dtype == np.uint16 else np.ascontiguousarray(a)).pin_memory()
    ps, pu, pv = pin(signs[2:]), pin(u[2:]), pin(v[2:])
    x = torch.from_numpy(make_x(1, g, 3).astype(np.float32)).cuda()
    side = torch.cuda.Stream()
    lay.load_blocks_async(2, ps, pu, pv, stream=side)
    ys = [busy.matmul(x) for _ in range(50)]          # main stream keeps working meanwhile
    ev = torch.cuda.Event()
    ev.record(side)
    torch.cuda.current_stream().wait_event(ev)
    assert lay.info()["n_active"] == 2                # a push never raises the active level
    lay.set_num_blocks(4)
    y = lay.matmul(x)
    torch.cuda.synchronize()
    xr = x.cpu().numpy().astype(np.float64)
    assert O.relative_l2(y.cpu().numpy().astype(np.float64), oracle_y(blocks, s32, 4, xr)) <= 1e-3
    assert all(torch.equal(a, ys[0]) for a in ys)


# ------------------------------------------------------------------ k > 16 (the paper's k ablation)
@pytest.mark.parametrize("k,dtype", [(32, "bf16"), (24, "bf16"), (32, "f32"), (20, "f16")])
def test_rank_above_16_every_path(bs, k, dtype):
    """k in (16, 32]: each block is held as two 16-rank halves sharing its sign tile; the
    decode kernels (e4m3 / fp16), the prefill path, the SIMT kernel, reconstruct and grouped
    calls all match the oracle on the same stored blocks."""
    d_out, d_in, n = 384, 640, 3
    g, s32, blocks = compress_case(d_out, d_in, n, dtype, 191 + k, k=k)
    lay = make_layer(bs, d_out, d_in, blocks, s32, dtype)
    assert lay.info()["k"] == k
    tol = 1e-5 if dtype == "f32" else 1e-3
    for batch in (1, 2, 3):
        x = make_x(batch, g, 30 + batch)
        for level in (1, n):
            lay.set_num_blocks(level)
            y, xr = gpu_y(lay, x)
            assert O.relative_l2(y, oracle_y(blocks, s32, level, xr)) <= tol, (batch, level)
    lay.set_num_blocks(n)
    w = lay.reconstruct(torch.float32).cpu().numpy().astype(np.float64)
    assert O.relative_l2(w, O.reconstruct(blocks, s32.astype(np.float64), n, d_out, d_in)) <= 1e-6
    x = make_x(40, g, 77)
    lay.set_kernel("simt")
    y, xr = gpu_y(lay, x[:2])
    assert O.relative_l2(y, oracle_y(blocks, s32, n, xr)) <= 1e-5
    if dtype == "bf16":
        lay.set_kernel("prefill")
        y, xr = gpu_y(lay, x, x_dtype=torch.bfloat16)
        assert O.relative_l2(y, oracle_y(blocks, s32, n, xr)) <= 1e-3
    lay.set_kernel("auto")
    if dtype != "f32":
        xs = [torch.from_numpy(make_x(1, g, 5).astype(np.float32)).cuda()]
        ys = bs.matmul_grouped([lay], xs)
        torch.cuda.synchronize()
        ref = oracle_y(blocks, s32, n, xs[0].cpu().numpy().astype(np.float64))
        assert O.relative_l2(ys[0].cpu().numpy().astype(np.float64), ref) <= 1e-3


# ------------------------------------------------------------------ mixed groups / graph capture
def test_grouped_mixed_ranks_and_graph_capture(bs):
    """A group mixing k = 16 and k = 32 members and different levels, captured into a CUDA
    graph and replayed: every member matches its individual call and the oracle."""
    g1, s1, b1 = compress_case(384, 512, 3, "bf16", 901)
    g2, s2, b2 = compress_case(256, 512, 2, "bf16", 902, k=32)
    l1 = make_layer(bs, 384, 512, b1, s1, "bf16")
    l2 = make_layer(bs, 256, 512, b2, s2, "bf16")
    l1.set_num_blocks(2)
    x = torch.from_numpy(make_x(2, g1, 3).astype(np.float32)).to(torch.bfloat16).cuda()
    y1 = torch.empty((2, 384), device="cuda")
    y2 = torch.empty((2, 256), device="cuda")
    grp = bs.Group([l1, l2], [x.data_ptr(), x.data_ptr()], [y1.data_ptr(), y2.data_ptr()])
    stream = torch.cuda.current_stream()
    grp(bs.BF16, bs.F32, 2, stream.cuda_stream)          # first call outside capture (workspaces)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.graph(graph, stream=cap):
        grp(bs.BF16, bs.F32, 2, cap.cuda_stream)
    stream.wait_stream(cap)
    y1.zero_()
    y2.zero_()
    graph.replay()
    torch.cuda.synchronize()
    xr = x.float().cpu().numpy().astype(np.float64)
    assert O.relative_l2(y1.cpu().numpy().astype(np.float64), oracle_y(b1, s1, 2, xr)) <= 1e-3
    assert O.relative_l2(y2.cpu().numpy().astype(np.float64), oracle_y(b2, s2, 2, xr)) <= 1e-3
    assert torch.equal(y1, l1.matmul(x)) or O.relative_l2(y1.cpu().numpy(), l1.matmul(x).cpu().numpy()) <= 1e-6


# ------------------------------------------------------------------ memory budget
@pytest.mark.parametrize("kind", ["average", "random", "greedy"])
def test_stackset_budget_walk(bs, kind):
    """A StackSet follows a shrinking then growing memory budget under each sorting:
    levels fit the budget (Average: differ by at most one), and every layer's y matches the
    oracle at its level."""
    from paper_2410_23918_b200.budget import StackSet
    shapes = [(256, 384), (384, 256), (200, 384)]
    cases = [compress_case(d_out, d_in, 4, "bf16", 1201 + j) for j, (d_out, d_in) in enumerate(shapes)]
    lays = [make_layer(bs, d_out, d_in, blocks, s32, "bf16") for (d_out, d_in), (g, s32, blocks) in zip(shapes, cases)]
    scores = [[0.3, 0.9, 0.2, 0.8], [0.1, 0.5, 0.6, 0.7], [0.4, 0.45, 0.95, 0.99]] if kind == "greedy" else None
    ss = StackSet(lays, order=[2, 0, 1] if kind == "average" else None, kind=kind, scores=scores, seed=3)
    full = sum(ss.sizes) * 4
    for frac in (1.0, 0.6, 0.3, 0.05, 0.45, 0.9):
        levels = ss.apply_budget(frac * full)
        if kind == "average":
            assert max(levels) - min(levels) <= 1
        assert sum(l * sz for l, sz in zip(levels, ss.sizes)) <= frac * full + 1e-6
        for lay, (g, s32, blocks), lv in zip(lays, cases, levels):
            assert lay.info()["n_active"] == lv
            y, xr = gpu_y(lay, make_x(1, g, 5))
            if lv == 0:
                assert not np.any(y)
            else:
                assert O.relative_l2(y, oracle_y(blocks, s32, lv, xr)) <= 1e-3


# ------------------------------------------------------------------ plain C use of the ABI
def test_c_demo_runs(bs, tmp_path):
    """examples/abi_demo.c (C99, host buffers, every level) agrees with its host reference."""
    import shutil
    import subprocess
    import os
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_2410_23918_b200")
    exe = tmp_path / "abi_demo"
    subprocess.run(["gcc", "-O2", "-std=c99", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "abi_demo.c"), "-L", lib_dir, "-lbitstack", "-lm",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr


# ------------------------------------------------------------------ H7: deterministic split-K
@pytest.mark.parametrize("dtype,batch", [("bf16", 1), ("bf16", 3), ("f32", 1), ("f32", 5)])
def test_split_k_reduction_is_deterministic(bs, dtype, batch):
    """Split-K partials are summed in CTA order by the last CTA of each row group (no float
    atomics): repeated calls give bitwise identical y, with many CTAs per row group."""
    g, s32, blocks = compress_case(512, 2048, 6, dtype, 131)
    lay = make_layer(bs, 512, 2048, blocks, s32, dtype)
    x = torch.from_numpy(make_x(batch, g, 17).astype(np.float32)).cuda()
    y0 = lay.matmul(x)
    for _ in range(20):
        assert torch.equal(lay.matmul(x), y0)
    torch.cuda.synchronize()
    ref = oracle_y(blocks, s32, 6, x.cpu().numpy().astype(np.float64))
    assert O.relative_l2(y0.cpu().numpy().astype(np.float64), ref) <= (1e-3 if dtype == "bf16" else 1e-5)


# ------------------------------------------------------------------ grouped decode launches
def _grouped_case(bs, shapes, seed):
    out = []
    for j, (d_out, d_in, n) in enumerate(shapes):
        g, s32, blocks = compress_case(d_out, d_in, n, "bf16", seed + 7 * j)
        out.append((g, s32, blocks, make_layer(bs, d_out, d_in, blocks, s32, "bf16")))
    return out


@pytest.mark.parametrize("batch", [1, 2, 3, 4, 7, 9])
def test_grouped_matches_individual_and_oracle(bs, batch):
    """bitstack_matmul_grouped: members of different shapes (ragged rows, ragged d_in) and
    levels run as ONE zq + ONE decode launch and give the individual calls' y (up to the
    order of the fp32 cross-CTA sums) and the oracle's within the decode tolerance."""
    case = _grouped_case(bs, [(512, 640, 4), (300, 200, 3), (1100, 264, 5), (128, 1000, 2)], 501)
    levels = [4, 1, 5, 2]
    for (_, _, _, lay), n in zip(case, levels):
        lay.set_num_blocks(n)
    xs = [torch.from_numpy(make_x(batch, g, 40 + batch).astype(np.float32)).to(torch.bfloat16).cuda()
          for g, _, _, _ in case]
    lays = [c[3] for c in case]
    c0 = bs.launch_count()
    ys = bs.matmul_grouped(lays, xs)
    torch.cuda.synchronize()
    if batch <= 5:   # one zq_mx_grouped + decode_mx_grouped pair; from 6 tokens each member's own path
        assert bs.launch_count() - c0 == 2
    for (g, s32, blocks, lay), n, x, y in zip(case, levels, xs, ys):
        y1 = lay.matmul(x)
        torch.cuda.synchronize()
        yg = y.cpu().numpy().astype(np.float64)
        assert O.relative_l2(yg, y1.cpu().numpy().astype(np.float64)) <= 1e-5
        ref = oracle_y(blocks, s32, n, x.float().cpu().numpy().astype(np.float64))
        assert O.relative_l2(yg, ref) <= 1e-3, (lay.rows, n)


def test_grouped_shared_x_more_ctas_than_sms(bs):
    """q/k/v-style members reading ONE x buffer; 4 members of 5120 rows need 160 row groups,
    more than one CTA per SM on 148 SMs (the decode kernel does not rely on co-residency)."""
    case = _grouped_case(bs, [(5120, 256, 2)] * 4, 611)
    g = case[0][0]
    x = torch.from_numpy(make_x(2, g, 3).astype(np.float32)).to(torch.bfloat16).cuda()
    lays = [c[3] for c in case]
    ys = bs.matmul_grouped(lays, [x] * 4, y_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    xr = x.float().cpu().numpy().astype(np.float64)
    for (_, s32, blocks, _), y in zip(case, ys):
        assert O.relative_l2(y.float().cpu().numpy().astype(np.float64), oracle_y(blocks, s32, 2, xr)) <= 4e-3


def test_grouped_fallbacks(bs):
    """Groups the fused launches cannot take (fp32 factors, prefill-size batches, a repeated
    handle, more than 8 members, n == 0) run member by member with identical results."""
    case = _grouped_case(bs, [(256, 384, 2), (384, 256, 3)], 701)
    g32, s32f, blocks32 = compress_case(200, 384, 2, "f32", 721)
    lay32 = make_layer(bs, 200, 384, blocks32, s32f, "f32")
    a, b = case[0][3], case[1][3]
    for batch in (1, 6, 20):
        xa = torch.from_numpy(make_x(batch, case[0][0], 9).astype(np.float32)).cuda()
        xb = torch.from_numpy(make_x(batch, case[1][0], 10).astype(np.float32)).cuda()
        for lays, xs in (([a, lay32, b], [xa, xa, xb]), ([a, a], [xa, xa]), ([b] * 9, [xb] * 9), ([a, b], [xa, xb])):
            ys = bs.matmul_grouped(lays, xs)
            torch.cuda.synchronize()
            for lay, x, y in zip(lays, xs, ys):
                y1 = lay.matmul(x)
                torch.cuda.synchronize()
                assert O.relative_l2(y.cpu().numpy().astype(np.float64), y1.cpu().numpy().astype(np.float64)) <= 1e-5
    a.set_num_blocks(0)
    ys = bs.matmul_grouped([a, b], [xa[:1], xb[:1]])
    torch.cuda.synchronize()
    assert not torch.any(ys[0])
    assert bs.matmul_grouped([], []) == []


@pytest.mark.parametrize("batch", [1, 3, 5])
def test_grouped_level_zero_members(bs, batch):
    """Members at level 0 (budgets below one level; the Random / Greedy sortings) get y = 0 and
    stay out of the fused launches; the others still run as ONE launch pair per <= 8 tokens."""
    case = _grouped_case(bs, [(512, 640, 3), (300, 200, 2), (1100, 264, 4), (128, 1000, 2)], 801)
    levels = [0, 2, 0, 1]
    for (_, _, _, lay), n in zip(case, levels):
        lay.set_num_blocks(n)
    lays = [c[3] for c in case]
    xs = [torch.from_numpy(make_x(batch, g, 60 + j).astype(np.float32)).to(torch.bfloat16).cuda()
          for j, (g, _, _, _) in enumerate(case)]
    ys = [torch.full((batch, l.rows), float("nan"), dtype=torch.float32, device="cuda") for l in lays]
    grp = bs.Group(lays, [x.data_ptr() for x in xs], [y.data_ptr() for y in ys])
    c0 = bs.launch_count()
    grp(bs.BF16, bs.F32, batch, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert bs.launch_count() - c0 == 2 * ((batch + 7) // 8)
    for (g, s32, blocks, lay), n, x, y in zip(case, levels, xs, ys):
        if n == 0:
            assert torch.count_nonzero(y) == 0          # NaN prefill overwritten by zeros
            continue
        xr = x.float().cpu().numpy().astype(np.float64)
        assert O.relative_l2(y.cpu().numpy().astype(np.float64), oracle_y(blocks, s32, n, xr)) <= 1e-3
    for _, _, _, lay in case:
        lay.set_num_blocks(0)
    ys2 = [torch.full_like(y, 1.0) for y in ys]       # every member at level 0: no launches at all
    c0 = bs.launch_count()
    bs.Group(lays, [x.data_ptr() for x in xs], [y.data_ptr() for y in ys2])(
        bs.BF16, bs.F32, batch, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert bs.launch_count() == c0 and all(torch.count_nonzero(y) == 0 for y in ys2)


# ------------------------------------------------------------------ H8: large-batch path
@pytest.mark.parametrize("shape", [(384, 640), (200, 296), (1100, 264), (128, 64)])
def test_prefill_parity_ragged(bs, shape):
    """Restored-tile GEMM path (prefill.cuh) forced at every batch: ragged rows (partial
    and odd row-tile counts), ragged d_in (chunk tails), batches across 256-token tiles,
    odd n (blocks per MMA step G = 2)."""
    d_out, d_in = shape
    g, s32, blocks = compress_case(d_out, d_in, 5, "bf16", 61 + d_out)
    lay = make_layer(bs, d_out, d_in, blocks, s32, "bf16")
    lay.set_kernel("prefill")
    c0 = bs.launch_count()
    gpu_y(lay, make_x(2, g, 1))
    assert bs.launch_count() - c0 == 4          # absmax + xprep + W' restore + gemm: the prefill kernels ran
    for batch in (1, 17, 256, 300, 600):
        x = make_x(batch, g, 300 + batch)
        for n in (1, 2, 5):
            lay.set_num_blocks(n)
            y, xr = gpu_y(lay, x, x_dtype=torch.bfloat16)
            err = O.relative_l2(y, oracle_y(blocks, s32, n, xr))
            assert err <= 1e-3, (batch, n, err)


def test_prefill_dtypes_auto_and_unsupported(bs):
    """AUTO picks the prefill path from batch 33 on (same y as forcing it); f32/bf16/f16
    activations; bf16 y (4e-3); fp32 factors refuse a forced prefill (E_UNSUPPORTED)."""
    g, s32, blocks = compress_case(256, 384, 4, "bf16", 71)
    lay = make_layer(bs, 256, 384, blocks, s32, "bf16")
    x = make_x(40, g, 9)
    c0 = bs.launch_count()
    y_auto, xr = gpu_y(lay, x)
    assert bs.launch_count() - c0 == 4
    assert O.relative_l2(y_auto, oracle_y(blocks, s32, 4, xr)) <= 1e-3
    lay.set_kernel("prefill")
    y_pf, _ = gpu_y(lay, x)
    np.testing.assert_array_equal(y_auto, y_pf)
    for xdt in (torch.float32, torch.bfloat16, torch.float16):
        y, xr = gpu_y(lay, x, x_dtype=xdt)
        assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 1e-3
    y, xr = gpu_y(lay, x, y_dtype=torch.bfloat16)
    assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 4e-3
    g32, s32f, blocks32 = compress_case(128, 256, 2, "f32", 72)
    lay32 = make_layer(bs, 128, 256, blocks32, s32f, "f32")
    x32 = make_x(64, g32, 1)
    y32, xr32 = gpu_y(lay32, x32)          # AUTO keeps the exact fp32-factor decode path
    assert O.relative_l2(y32, oracle_y(blocks32, s32f, 2, xr32)) <= 1e-5
    lay32.set_kernel("prefill")
    with pytest.raises(bs.BitStackError) as e:
        gpu_y(lay32, x32)
    assert e.value.name == "E_UNSUPPORTED"


# ------------------------------------------------------------------ full sizes, sampled rows
def _sampled_reference(signs, u, v, s, n, x, rows, d_out, d_in):
    """Oracle y on a subset of output rows: slice the stored blocks' rows (oracle unpack
    / pack) and run the dense oracle on the slice."""
    sub = []
    for i in range(n):
        sm = O.unpack_signs(signs[i], d_out, d_in)[rows]
        sub.append(O.Block(signs=O.pack_signs(sm), u=np.asarray(u[i][rows], np.float64),
                           v=np.asarray(v[i], np.float64)))
    return O.matmul_dense(sub, s.astype(np.float64), n, x)


@pytest.mark.parametrize("name,d_out,d_in,n,batch", [
    ("c5_down_70b", 8192, 28672, 12, 1),
    ("c5_down_70b_b4", 8192, 28672, 12, 4),
    ("c3_up", 14336, 4096, 8, 16),
    ("c3_gate_prefill", 14336, 4096, 8, 2048),
    ("c3_down_prefill", 4096, 14336, 8, 300),
    ("c4_kproj", 1024, 4096, 3, 1),
])
def test_full_size_sampled_rows(bs, name, d_out, d_in, n, batch):
    """Full BASELINE shapes (random stored-form blocks from synthetic/): the GPU's y on
    96 sampled rows equals the oracle's, <= 1e-3."""
    signs, u32, v32, s = make_random_blocks(n, d_out, d_in, 16, seed=seed_for(5, 1, "blocks"))
    ub = O.bf16_bits(u32)
    vb = O.bf16_bits(v32)
    u_val = O.round_to_dtype(u32, "bf16")
    v_val = O.round_to_dtype(v32, "bf16")
    lay = bs.Layer(d_out, d_in, k=16, n_capacity=n, factor_dtype="bf16")
    lay.load_blocks(0, signs, ub, vb, s)
    g = channel_gains(d_in, seed_for(5, 1, "gains"))
    x = make_x(batch, g, 3)
    y, xr = gpu_y(lay, x, x_dtype=torch.bfloat16)
    rows = np.sort(np.random.default_rng(1).choice(d_out, 96, replace=False))
    ref = _sampled_reference(signs, u_val, v_val, s, n, xr, rows, d_out, d_in)
    assert O.relative_l2(y[:, rows], ref) <= 1e-3
    del lay


# ------------------------------------------------------------------ on-disk block store
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_store_load_range_matches_memory_load(bs, tmp_path, dtype):
    """Blocks written to a BSTK file (two stacks interleaved, as the universal order does) and
    streamed back with bitstack_store_load_range give the same y as bitstack_load_blocks from
    memory, bit for bit, and a partial record range is a usable prefix (P:8 "basic transmission
    units")."""
    cases = [compress_case(384, 512, 4, dtype, 7100), compress_case(256, 640, 4, dtype, 7101)]
    path = str(tmp_path / "m.bstk")
    with bs.Store.create(path) as st:
        for i in range(4):
            for sid, (g, s32, blocks) in enumerate(cases):
                signs, u, v = stack_blocks(blocks[i:i + 1], dtype)
                st.append(sid, i, signs[0], u[0], v[0], s32 if i == 0 else None, factor_dtype=dtype)
    with bs.Store.open(path) as st:
        for sid, (g, s32, blocks) in enumerate(cases):
            d_out, d_in = (384, 512) if sid == 0 else (256, 640)
            ref_lay = make_layer(bs, d_out, d_in, blocks, s32, dtype)
            lay = bs.Layer(d_out, d_in, k=16, n_capacity=4, factor_dtype=dtype)
            x = make_x(3, g, 11)
            for i in range(4):                     # record of (stack sid, block i) = 2 i + sid
                st.load_range(lay, 2 * i + sid, 1)
                lay.set_num_blocks(i + 1)
                ref_lay.set_num_blocks(i + 1)
                y, xr = gpu_y(lay, x)
                y_ref, _ = gpu_y(ref_lay, x)
                assert np.array_equal(y, y_ref)
                assert O.relative_l2(y, oracle_y(blocks, s32, i + 1, xr)) <= 1e-3
            with pytest.raises(bs.BitStackError):   # a record of the other stack: shape mismatch
                st.load_range(lay, 1 - sid, 1)
    # one stack, contiguous: a 2-record prefix then the rest
    g, s32, blocks = cases[0]
    path2 = str(tmp_path / "one.bstk")
    with bs.Store.create(path2) as st:
        signs, u, v = stack_blocks(blocks, dtype)
        for i in range(4):
            st.append(0, i, signs[i], u[i], v[i], s32 if i == 0 else None, factor_dtype=dtype)
    with bs.Store.open(path2) as st:
        lay = bs.Layer(384, 512, k=16, n_capacity=4, factor_dtype=dtype)
        st.load_range(lay, 0, 2)
        torch.cuda.synchronize()
        assert lay.info()["n_resident"] == 2
        lay.set_num_blocks(2)                      # loads never raise the active level
        x = make_x(2, g, 12)
        y, xr = gpu_y(lay, x)
        assert O.relative_l2(y, oracle_y(blocks, s32, 2, xr)) <= 1e-3
        st.load_range(lay, 2, 2)
        lay.set_num_blocks(4)
        y, xr = gpu_y(lay, x)
        assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 1e-3


# ------------------------------------------------------------------ restore-and-multiply path
@pytest.mark.parametrize("shape", [(256, 384, 3, 16, "bf16"), (300, 520, 5, 16, "bf16"), (1100, 264, 2, 16, "f16"),
                                   (128, 1000, 4, 32, "bf16"), (640, 640, 17, 16, "bf16")])
@pytest.mark.parametrize("batch", [1, 3, 8, 16, 17, 32])
def test_rgemv_parity_ragged(bs, shape, batch):
    """bitstack_matmul through the restore-and-multiply kernel (W' restored per 128 x 128 unit in
    the SM, y += W' X'^T in tf32) against the oracle: ragged rows / d_in, k = 32 halves, fp16
    factors, n above the prefill's 16, batch 1..32 (both token paddings, 16 and 32)."""
    d_out, d_in, n, k, dt = shape
    g, s32, blocks = compress_case(d_out, d_in, n, dt, 9300 + d_out + n, k=k)
    lay = make_layer(bs, d_out, d_in, blocks, s32, dt)
    lay.set_kernel("rgemv")
    x = make_x(batch, g, 60 + batch)
    c0 = bs.launch_count()
    y, xr = gpu_y(lay, x)
    assert bs.launch_count() - c0 == 2            # rg_xprep + rgemv
    assert O.relative_l2(y, oracle_y(blocks, s32, n, xr)) <= 1e-3
    for lvl in (1, max(1, n // 2)):               # lower levels of the same stack
        lay.set_num_blocks(lvl)
        y, xr = gpu_y(lay, x)
        assert O.relative_l2(y, oracle_y(blocks, s32, lvl, xr)) <= 1e-3


def test_rgemv_dispatch_bf16_y_and_determinism(bs):
    """AUTO: the e4m3 decode up to 5 tokens (zq + decode), restore-and-multiply for 6..32 (xprep +
    rgemv), the prefill above (4 launches); forced rgemv gives bf16 y within the bf16-y bar and
    bitwise identical repeated calls, and refuses more than 32 tokens (E_UNSUPPORTED)."""
    g, s32, blocks = compress_case(512, 768, 4, "bf16", 9400)
    lay = make_layer(bs, 512, 768, blocks, s32, "bf16")
    for batch, launches in [(5, 2), (6, 2), (32, 2), (33, 4)]:
        x = make_x(batch, g, 70 + batch)
        c0 = bs.launch_count()
        y, xr = gpu_y(lay, x)
        assert bs.launch_count() - c0 == launches, batch
        assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 1e-3
    lay.set_kernel("rgemv")
    x = make_x(12, g, 80)
    y, xr = gpu_y(lay, x, y_dtype=torch.bfloat16)
    assert O.relative_l2(y, oracle_y(blocks, s32, 4, xr)) <= 4e-3
    y1, _ = gpu_y(lay, x)
    for _ in range(5):
        y2, _ = gpu_y(lay, x)
        assert np.array_equal(y1, y2)
    with pytest.raises(bs.BitStackError) as e:
        gpu_y(lay, make_x(33, g, 81))
    assert e.value.name == "E_UNSUPPORTED"
    # CUDA-graph capture of a warmed-up call, replayed: same bytes as the eager call
    xg = torch.from_numpy(x.astype(np.float32)).cuda()
    yg = torch.empty((12, 512), dtype=torch.float32, device="cuda")
    lay.matmul_raw(xg.data_ptr(), bs.F32, yg.data_ptr(), bs.F32, 12, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    y_eager = yg.clone()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cap):
        lay.matmul_raw(xg.data_ptr(), bs.F32, yg.data_ptr(), bs.F32, 12, cap.cuda_stream)
    yg.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, y_eager)


# ------------------------------------------------------------------ output bounds (guard bands)
@pytest.mark.parametrize("kernel,batch,dtype", [("auto", 1, "bf16"), ("auto", 3, "bf16"), ("auto", 8, "f16"),
                                                ("auto", 20, "bf16"), ("rgemv", 5, "bf16"), ("simt", 2, "bf16"),
                                                ("auto", 2, "f32")])
def test_outputs_stay_inside_y(bs, kernel, batch, dtype):
    """Every path writes exactly y[batch][rows_local]: guard bands of NaN before and after y in the
    same allocation come back untouched (compute-sanitizer is not available on the GPU pool, so
    out-of-bounds writes are checked this way), and y itself matches the oracle."""
    g, s32, blocks = compress_case(300, 392, 3, dtype, 9500 + batch)
    lay = make_layer(bs, 300, 392, blocks, s32, dtype)
    if kernel != "auto":
        lay.set_kernel(kernel)
    guard = 4096
    buf = torch.full((guard + batch * 300 + guard,), float("nan"), dtype=torch.float32, device="cuda")
    y = buf[guard:guard + batch * 300].view(batch, 300)
    x = torch.from_numpy(make_x(batch, g, 90).astype(np.float32)).cuda()
    lay.matmul_raw(x.data_ptr(), bs.F32, y.data_ptr(), bs.F32, batch, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.isnan(buf[:guard]).all() and torch.isnan(buf[guard + batch * 300:]).all()
    ref = oracle_y(blocks, s32, 3, x.double().cpu().numpy())
    assert O.relative_l2(y.double().cpu().numpy(), ref) <= (1e-5 if dtype == "f32" else 1e-3)


def test_prefill_more_than_16_blocks(bs):
    """The prefill's W' restore runs on the restore-and-multiply pipeline, which has no block-count
    limit: 20 blocks (and 12 k = 32 blocks = 24 halves) at 40 tokens take the prefill path and
    match the oracle."""
    for (d_out, d_in, n, k) in [(384, 512, 20, 16), (256, 384, 12, 32)]:
        g, s32, blocks = compress_case(d_out, d_in, n, "bf16", 9700 + n, k=k)
        lay = make_layer(bs, d_out, d_in, blocks, s32, "bf16")
        x = make_x(40, g, 91)
        c0 = bs.launch_count()
        y, xr = gpu_y(lay, x)
        assert bs.launch_count() - c0 == 4          # absmax + xprep + W' restore + GEMM
        assert O.relative_l2(y, oracle_y(blocks, s32, n, xr)) <= 1e-3


def test_prefill_register_product_restore_variant():
    """The opt-in W' restore with the products in registers (BS_WRESTORE_HMMA=1, csrc/wrestore.cuh)
    passes the prefill parity tests too (a fresh process: the switch is read once per process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BS_WRESTORE_HMMA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "tests/test_gpu_parity.py",
                        "-k", "prefill_parity_ragged or prefill_more_than or prefill_dtypes"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_rgemv_hybrid_register_products_variant():
    """The opt-in restore-and-multiply / W' restore variant whose channel half 1 forms its products
    with mma.sync in registers (BS_RG_HYB=1) passes the rgemv and prefill parity tests (fresh process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BS_RG_HYB="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "tests/test_gpu_parity.py",
                        "-k", "rgemv_parity or prefill_parity_ragged or prefill_more_than"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
