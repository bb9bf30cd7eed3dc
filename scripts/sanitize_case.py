"""Small calls through every GPU path, for compute-sanitizer (memcheck / racecheck / synccheck):
MX decode (B = 1, 3, k = 32 fused halves), fp16 decode (fp32 factors), prefill (B = 20), grouped
launch, reconstruct, load from a block store.  Checks y against the oracle at the end so that a
sanitizer run also shows the results were right."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_2410_23918_b200 as pkg
from bitstack_test_helpers import stack_blocks
from oracle import bitstack_oracle as O
from synthetic import channel_gains, make_calibration, make_weight, make_x

pkg.load_library()
worst = 0.0


def case(d_out, d_in, n, dt, k=16, seed=1):
    g = channel_gains(d_in, seed + 4)
    s, blocks = O.compress(make_weight(d_out, d_in, seed), make_calibration(256, g, seed + 1), n, k, dtype=dt,
                           method="exact", seed=seed)
    signs, u, v = stack_blocks(blocks, dt)
    lay = pkg.Layer(d_out, d_in, k=k, n_capacity=n, factor_dtype=dt)
    lay.load_blocks(0, signs, u, v, s.astype(np.float32))
    return g, s.astype(np.float32), blocks, lay


def check(lay, g, s, blocks, batch, seed):
    global worst
    x = torch.from_numpy(make_x(batch, g, seed).astype(np.float32)).cuda()
    y = lay.matmul(x)
    torch.cuda.synchronize()
    ref = O.matmul_dense(blocks, s.astype(np.float64), lay.info()["n_active"], x.double().cpu().numpy())
    worst = max(worst, O.relative_l2(y.double().cpu().numpy(), ref))


g, s, blocks, lay = case(256, 512, 3, "bf16")
for b in (1, 3):
    check(lay, g, s, blocks, b, 10 + b)
check(lay, g, s, blocks, 20, 30)                     # prefill
lay.reconstruct()
g2, s2, blocks2, lay2 = case(128, 256, 2, "f32", seed=2)
check(lay2, g2, s2, blocks2, 2, 40)                  # fp16 decode (fp32 factors)
g3, s3, blocks3, lay3 = case(256, 384, 2, "bf16", k=32, seed=3)
check(lay3, g3, s3, blocks3, 1, 50)                  # fused k = 32 halves
xs = [torch.from_numpy(make_x(2, g, 60).astype(np.float32)).cuda(),
      torch.from_numpy(make_x(2, g, 61).astype(np.float32)).cuda()]
g4, s4, blocks4, lay4 = case(256, 512, 2, "bf16", seed=4)
ys = pkg.matmul_grouped([lay, lay4], xs)            # grouped launch
torch.cuda.synchronize()
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "m.bstk")
    sg, uu, vv = stack_blocks(blocks, "bf16")
    with pkg.Store.create(path) as st:
        for i in range(3):
            st.append(0, i, sg[i], uu[i], vv[i], s if i == 0 else None, factor_dtype="bf16")
    lay5 = pkg.Layer(256, 512, k=16, n_capacity=3, factor_dtype="bf16")
    with pkg.Store.open(path) as st:
        st.load_range(lay5, 0, 3)
    lay5.set_num_blocks(3)
    check(lay5, g, s, blocks, 2, 70)
print(f"sanitize_case: all paths ran; worst relative L2 vs oracle {worst:.2e}")
assert worst <= 1e-3
