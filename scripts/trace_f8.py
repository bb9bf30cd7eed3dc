"""Timeline of CTA 0 of the e4m3 decode kernel (C2 shape, n=16, B=1) via the debug hook."""
import ctypes, os, sys
sys.path.insert(0, ".")
from paper_2410_23918_b200.build import build
if "BITSTACK_LIB" not in os.environ:
    os.environ["BITSTACK_LIB"] = build(extra=["-DBS_DECODE_TRACE"], out=os.path.abspath("scripts/libbitstack_trace.so"))
import numpy as np, torch
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
tr = torch.zeros(65536 + 4 * 1024, dtype=torch.int64, device="cuda")
lib.bitstack_debug_set(tr.data_ptr(), None)
lay.matmul(x); torch.cuda.synchronize()
lib.bitstack_debug_set(None, None)
full = tr.cpu().numpy()
t = full[:65536].reshape(-1, 16)
cta = full[65536:].reshape(-1, 4)
cta = cta[cta[:, 0] != 0]
if len(cta):
  t0 = cta[:, 0].min()
  print('CTAs', len(cta), 'entry spread us', (cta[:, 0].max() - t0) / 1e3, 'exit (wg3 done) min/med/max us', (cta[:, 1].min() - t0) / 1e3, (np.median(cta[:, 1]) - t0) / 1e3, (cta[:, 1].max() - t0) / 1e3, 'units min/max', cta[:, 2].min(), cta[:, 2].max())
if os.environ.get("BS_DECODE_WG") != "1":
    print("unit | warpgroup 3 waiter warp: before_go go_done sttm_issued st_done loop_end | issuer: before_sync synced issued")
    for k in range(28):
        print(k, *[f"{x:6d}" for x in t[k, :5]], "|", *[f"{x:6d}" for x in t[k, 8:11]])
    sys.exit(0)
print("nonzero", int((t != 0).sum()), "max", int(t.max()), "min", int(t.min()))
nu = int((t[:, 6] != 0).sum())
print("units traced:", nu)
print("unit  loop_head  full_ok  slot_ok  bar1_done  sttm_issued  wait_st_done  bar2_done  mma0 mma1 mma2 mma3 mma_issued  (warpgroup 3)")
for k in range(min(nu, 40)):
    print(k, *[f"{x:6d}" for x in t[k, [7, 2, 0, 1, 3, 4, 5, 12, 13, 14, 15, 6]]])
