"""Per-unit timeline of CTA 0 of one decode_mx call (trace build -DBS_MX_TRACE) plus the CTA
entry / exit spread.  Usage: python scripts/mx_trace.py [c2|c5] [nomma]"""
import ctypes, os, sys
sys.path.insert(0, ".")
from paper_2410_23918_b200.build import build
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
extra = ["-DBS_MX_TRACE"] + (["-DBS_MX_EXP_NOST", "-DBS_MX_EXP_NOMMA", "-DBS_MX_EXP_NOEXP"] if "skel" in sys.argv else [])
os.environ["BITSTACK_LIB"] = build(extra=extra, out=os.path.abspath("scripts/variants/lib_trace%s.so" % ("_skel" if "skel" in sys.argv else "")))
import numpy as np, torch
import paper_2410_23918_b200 as pkg
from paper_2410_23918_b200 import bitstack as B
from synthetic import make_random_blocks, channel_gains, make_x
n, do, di = (16, 4096, 4096) if wl == "c2" else (12, 8192, 28672)
signs, u, v, s = make_random_blocks(n, do, di, 16, seed=5)
ncp = 6 if wl == "c2" else 2
lays = []
for i in range(ncp):
    lay = pkg.Layer(do, di, 16, n, "bf16")
    lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
    lays.append(lay)
for a in sys.argv:
    if a.startswith("n="):
        for l in lays: l.set_num_blocks(int(a[2:]))
x = torch.from_numpy(make_x(1, channel_gains(di, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
y = torch.empty(1, do, device="cuda")
for _ in range(5):
    for l in lays: l.matmul(x, y)
torch.cuda.synchronize()
lib = B.load_library(); lib.bitstack_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for rep in range(2):
    tr = torch.zeros(65536 + 4 * 1024, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.bitstack_debug_set(tr.data_ptr(), None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); lays[rep % ncp].matmul(x, y); e1.record(); torch.cuda.synchronize()
    lib.bitstack_debug_set(None, None)
    full = tr.cpu().numpy()
    cta = full[65536:].reshape(-1, 4)
    cta = cta[cta[:, 0] != 0]
    t0 = cta[:, 0].min()
    ex = np.sort((cta[:, 1] - t0) / 1e3)
    ent = np.sort((cta[:, 0] - t0) / 1e3)
    print("entry quantiles us", np.round(ent[[0, len(ent)//4, len(ent)//2, 3*len(ent)//4, -1]], 2))
    print(f"call {e0.elapsed_time(e1)*1e3:.1f} us; CTAs {len(cta)} entry spread {(cta[:,0].max()-t0)/1e3:.2f} us; exit min {ex[0]:.2f} med {np.median(ex):.2f} max {ex[-1]:.2f} us; units {cta[:,2].min()}-{cta[:,2].max()}")
t = full[:65536].reshape(-1, 16)
print("unit | prod_issue | exp0: landed expanded afull_arrive st_done | iss: afull_done - commit | iss: loop_top - -  (cycles, CTA clock)")
nu = int(cta[0, 2])
for k in list(range(min(nu, 24))) + list(range(max(24, nu - 6), nu)):
    print(f"{k:4d}", *[f"{x:7d}" for x in t[k, :11]])
d = np.diff(t[:nu, 7])
print("mma commit interval median", np.median(d[2:]) if len(d) > 3 else None)
