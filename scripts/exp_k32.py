"""Batch-1 decode time for k = 16 vs k = 32 (C2 shape, n = 16; layer copies rotated > L2)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2410_23918_b200 as pkg
from synthetic import make_random_blocks, channel_gains, make_x
pkg.load_library()
d, n = 4096, 16
x = torch.from_numpy(make_x(1, channel_gains(d, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
for k in (16, 32):
    signs, u, v, s = make_random_blocks(n, d, d, k, seed=5)
    lays = []
    for c in range(4):
        lay = pkg.Layer(d, d, k, n, "bf16")
        lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
        lays.append(lay)
    y = torch.empty(1, d, device="cuda")
    for _ in range(10):
        for l in lays: l.matmul(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(200): lays[i % 4].matmul(x, y)
    e1.record(); torch.cuda.synchronize()
    print(f"k={k}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us per call (eager)")
    del lays
