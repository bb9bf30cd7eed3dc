"""Eager bitstack_matmul calls of one bench workload shape (for ncu launch lists):
python scripts/call_once.py c2|c5 n=<blocks> calls=<k> batch=<b>"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2410_23918_b200 as pkg
from synthetic import make_random_blocks, channel_gains, make_x
args = dict(a.split("=") for a in sys.argv[2:])
wl = sys.argv[1]
n_all, do, di = (16, 4096, 4096) if wl == "c2" else (12, 8192, 28672)
n = int(args.get("n", n_all))
calls = int(args.get("calls", 10))
batch = int(args.get("batch", 1))
signs, u, v, s = make_random_blocks(n_all, do, di, 16, seed=5)
lay = pkg.Layer(do, di, 16, n_all, "bf16")
lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
lay.set_num_blocks(n)
x = torch.from_numpy(make_x(batch, channel_gains(di, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
y = torch.empty(batch, do, device="cuda")
for _ in range(calls):
    lay.matmul(x, y)
torch.cuda.synchronize()
print("ok")
