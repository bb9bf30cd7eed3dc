"""Per-stage timeline of CTA 0 of one rgemv call (trace build -DBS_RG_TRACE): producer issue /
publish, MMA warp full-seen / issue, restore warps 0 and last: P seen / done (cycles)."""
import ctypes, os, sys
sys.path.insert(0, ".")
from paper_2410_23918_b200.build import build
extra = ["-DBS_RG_TRACE"] + [a for a in sys.argv[1:] if a.startswith("-D")]
os.environ["BITSTACK_LIB"] = build(extra=extra, out=os.path.abspath("scripts/variants/lib_rgtrace.so"))
import numpy as np, torch
import paper_2410_23918_b200 as pkg
from paper_2410_23918_b200 import bitstack as B
from synthetic import make_random_blocks, channel_gains, make_x
n, do, di = 16, 4096, 4096
signs, u, v, s = make_random_blocks(n, do, di, 16, seed=5)
lay = pkg.Layer(do, di, 16, n, "bf16")
lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
lay.set_kernel("rgemv")
x = torch.from_numpy(make_x(8, channel_gains(di, 5), 6).astype(np.float32)).cuda()
for _ in range(3):
    y = lay.matmul(x)
torch.cuda.synchronize()
lib = B.load_library(); lib.bitstack_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
tr = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
lib.bitstack_debug_set(tr.data_ptr(), None)
y = lay.matmul(x)
torch.cuda.synchronize()
lib.bitstack_debug_set(None, None)
t = tr.cpu().numpy().reshape(-1, 8)
T = int((t[:, 2] != 0).sum())
t0 = t[0, 0]
t = t[:T] - t0
print("stage | prod_issue r0_ld_done | mma_full mma_issue | r0_P r0_done | rL_P rL_done   (cycles from stage 0 issue)")
for k in list(range(min(T, 40))) + list(range(max(40, T - 8), T)):
    print(f"{k:4d}", *[f"{v:8d}" for v in t[k]])
d = np.diff(t[:, 3])
print("MMA issue interval median", np.median(d[8:]), "; restore warp0 per-stage median", np.median(np.diff(t[:, 5])[8:]))
print("median lags: mma_full-issue", np.median(t[8:, 2] - t[8:, 0]),
      " mma_issue-full", np.median(t[8:, 3] - t[8:, 2]), " r0_P-mma_issue", np.median(t[8:, 4] - t[8:, 3]),
      " r0 P->ld done", np.median(t[8:, 1] - t[8:, 4]), " r0 ld done->done", np.median(t[8:, 5] - t[8:, 1]),
      " r0 done->next P", np.median(t[9:, 4] - t[8:-1, 5]))
