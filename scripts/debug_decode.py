"""Debug harness for the tcgen05 decode kernel: dumps CTA 0's on-chip Z tile and
raw TMEM accumulators via the bitstack_debug_set test hook and compares them
with a numpy emulation of what they should hold.  Not part of the product."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2410_23918_b200 as pkg  # noqa: E402
from paper_2410_23918_b200 import bitstack as B  # noqa: E402


def run(d_out, d_in, n, signs, u, v, s, x, dtype="f32"):
    lib = B.load_library()
    lay = pkg.Layer(d_out, d_in, k=16, n_capacity=n, factor_dtype=dtype)
    lay.load_blocks(0, signs, u, v, s)
    N = 16 * (2 if dtype == "f32" else 1)
    acc = torch.full((8 * 128 * N + 128 * 16 + 1,), float("nan"), device="cuda")
    z = torch.zeros((128 * N * 2 // 4,), dtype=torch.int32, device="cuda")
    lib.bitstack_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.bitstack_debug_set(acc.data_ptr(), z.data_ptr())
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    y = lay.matmul(xt)
    torch.cuda.synchronize()
    lib.bitstack_debug_set(None, None)
    zb = z.cpu().numpy().view(np.uint8)
    zz = np.zeros((N, 128), np.float32)
    for nn in range(N):
        for k in range(128):
            off = ((k // 8) * (N // 8) + nn // 8) * 128 + (nn % 8) * 16 + (k % 8) * 2
            zz[nn, k] = zb[off:off + 2].view(np.float16)[0]
    a = acc.cpu().numpy()
    araw = a[8 * 128 * N:8 * 128 * N + 128 * 16].view(np.uint32).reshape(128, 16)
    print("  A readback row0:", [hex(int(q)) for q in araw[0, :6]], " row 33:", [hex(int(q)) for q in araw[33, :4]],
          " tbase:", hex(int(a[-1:].view(np.uint32)[0])))
    return y.cpu().numpy(), zz, a[:8 * 128 * N].reshape(8, 128, N)


def main():
    d_out = d_in = 128
    n = 1
    signs = np.full((1, d_out * d_in // 8), 0xFF, np.uint8)
    u = np.zeros((1, d_out, 16), np.float32)
    v = np.zeros((1, d_in, 16), np.float32)
    u[0, :, 0] = 1.0
    v[0, :, 0] = 1.0
    s = np.ones(d_in, np.float32)
    x = np.ones((1, d_in), np.float32)
    for dtype in ("bf16", "f32"):
        uu = u if dtype == "f32" else torch.from_numpy(u).to(torch.bfloat16)
        vv = v if dtype == "f32" else torch.from_numpy(v).to(torch.bfloat16)
        y, zz, acc = run(d_out, d_in, n, signs, uu, vv, s, x, dtype)
        print(dtype, "y[:4] =", y[0, :4], "(expect 128)")
        print("  Z row 0 [:8] =", zz[0, :8], " Z row1 [:4] =", zz[1, :4], " nan in Z:", np.isnan(zz).sum())
        print("  acc tile0 row0 [:18] =", acc[0, 0, :18])
        print("  acc tile0 row5 [:4] =", acc[0, 5, :4], " nan count tile0:", np.isnan(acc[0]).sum())
    # random case: compare Z and T with numpy
    rng = np.random.default_rng(0)
    signs = rng.integers(0, 256, (1, d_out * d_in // 8), dtype=np.uint8)
    v = rng.standard_normal((1, d_in, 16)).astype(np.float32)
    u = rng.standard_normal((1, d_out, 16)).astype(np.float32)
    x = rng.standard_normal((1, d_in)).astype(np.float32)
    y, zz, acc = run(d_out, d_in, 1, signs, u, v, s, x, "f32")
    e = np.floor(np.log2(256.0 / np.abs(v[0]).max(axis=0)))
    vp = v[0] * 2.0 ** e
    z_ref = (vp * x[0][:, None])  # [c, r]
    S = np.where(np.unpackbits(signs[0], bitorder="little").reshape(d_out, d_in) == 1, 1.0, -1.0)
    t_ref = S @ z_ref
    print("random: Z hi err", np.abs(zz[:16].T - z_ref).max(), " T err", np.nanmax(np.abs(acc[0, :, :16] + acc[0, :, 16:32] - t_ref)))
    print("  T ref row0[:4]", t_ref[0, :4], " got", acc[0, 0, :4] + acc[0, 0, 16:20])
    y_ref = x[0] @ (S * (u[0] @ v[0].T)).T
    print("  y err", np.abs(y[0] - y_ref).max() / np.abs(y_ref).max())


if __name__ == "__main__":
    main()
