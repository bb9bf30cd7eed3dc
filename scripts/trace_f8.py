"""Timeline of CTA 0 of the e4m3 decode kernel (C2 shape, n=16, B=1) via the debug hook."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2410_23918_b200 as pkg
from paper_2410_23918_b200 import bitstack as B
from synthetic import make_random_blocks, channel_gains, make_x
n, d = 16, 4096
signs, u, v, s = make_random_blocks(n, d, d, 16, seed=5)
lay = pkg.Layer(d, d, 16, n, "bf16")
lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
x = torch.from_numpy(make_x(1, channel_gains(d, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
for _ in range(3): lay.matmul(x)
lib = B.load_library(); lib.bitstack_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
tr = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib.bitstack_debug_set(tr.data_ptr(), None)
lay.matmul(x); torch.cuda.synchronize()
lib.bitstack_debug_set(None, None)
t = tr.cpu().numpy().reshape(-1, 8)
print("nonzero", int((t != 0).sum()), "max", int(t.max()), "min", int(t.min()))
nu = int((t[:, 0] != 0).sum())
print("units traced:", nu)
print("unit  prod_issue  exp_full  exp_a_empty_ok  exp_sttm_issued  exp_wait_st_done  exp_arrive  mma_full  mma_issued")
for k in range(min(nu, 40)):
    print(k, *[f"{x:9d}" for x in t[k, [0, 1, 2, 6, 7, 3, 4, 5]]])
