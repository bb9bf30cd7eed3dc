"""Debug the e4m3 decode kernel on small cases: compare y with the oracle for several shapes/batches."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2410_23918_b200 as pkg
from oracle import bitstack_oracle as O
from synthetic import channel_gains, make_calibration, make_weight, make_x

def case(d_out, d_in, n, batch, seed=1):
    g = channel_gains(d_in, seed + 4)
    w = make_weight(d_out, d_in, seed)
    s, blocks = O.compress(w, make_calibration(max(256, d_in), g, seed + 1), n, 16, dtype="bf16", seed=seed)
    s32 = s.astype(np.float32)
    signs = np.stack([b.signs for b in blocks])
    u = O.bf16_bits(np.stack([b.u for b in blocks])); v = O.bf16_bits(np.stack([b.v for b in blocks]))
    lay = pkg.Layer(d_out, d_in, k=16, n_capacity=n, factor_dtype="bf16")
    lay.load_blocks(0, signs, u, v, s32)
    x = torch.from_numpy(make_x(batch, g, 3).astype(np.float32)).cuda()
    for kern in ("tc", "simt"):
        lay.set_kernel(kern)
        y = lay.matmul(x).cpu().numpy()
        ref = O.matmul_dense(blocks, s32.astype(np.float64), n, x.cpu().numpy().astype(np.float64))
        err = [O.relative_l2(y[b:b+1], ref[b:b+1]) for b in range(batch)]
        print(f"{d_out}x{d_in} n={n} B={batch} {kern}: rel per batch {np.array(err)}  y0[:3]={y[0,:3]} ref0[:3]={ref[0,:3]}")

for args in [(128, 128, 1, 1), (256, 256, 1, 1), (128, 256, 2, 1), (384, 640, 5, 1), (384, 640, 5, 2), (1024, 512, 2, 1), (1152, 256, 1, 1)]:
    case(*args)
