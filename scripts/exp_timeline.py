"""Single-call timeline of the C2 decode pair: event time of one eager call, the CTA entry /
exit spread from the trace build, and per-unit timestamps of CTA 0 (scripts/trace_f8.py)."""
import ctypes, os, sys
sys.path.insert(0, ".")
from paper_2410_23918_b200.build import build
os.environ["BITSTACK_LIB"] = build(extra=["-DBS_DECODE_TRACE"], out=os.path.abspath("scripts/libbitstack_trace.so"))
import numpy as np, torch
import paper_2410_23918_b200 as pkg
from paper_2410_23918_b200 import bitstack as B
from synthetic import make_random_blocks, channel_gains, make_x
n, d = 16, 4096
signs, u, v, s = make_random_blocks(n, d, d, 16, seed=5)
lays = []
for i in range(6):   # rotate over copies (> L2)
    lay = pkg.Layer(d, d, 16, n, "bf16")
    lay.load_blocks(0, signs, torch.from_numpy(u).to(torch.bfloat16), torch.from_numpy(v).to(torch.bfloat16), s)
    lays.append(lay)
x = torch.from_numpy(make_x(1, channel_gains(d, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
y = torch.empty(1, d, device="cuda")
for _ in range(5):
    for l in lays: l.matmul(x, y)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for k in range(60): lays[k % 6].matmul(x, y)
    e1.record(); torch.cuda.synchronize()
    print("eager us/call", e0.elapsed_time(e1) / 60 * 1e3)
lib = B.load_library(); lib.bitstack_debug_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for rep in range(3):
    tr = torch.zeros(65536 + 4 * 1024, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib.bitstack_debug_set(tr.data_ptr(), None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); lays[rep].matmul(x, y); e1.record(); torch.cuda.synchronize()
    lib.bitstack_debug_set(None, None)
    full = tr.cpu().numpy()
    cta = full[65536:].reshape(-1, 4)
    cta = cta[cta[:, 0] != 0]
    t0 = cta[:, 0].min()
    ex = np.sort((cta[:, 1] - t0) / 1e3)
    print(f"call {e0.elapsed_time(e1)*1e3:.1f} us; CTAs {len(cta)} entry spread {(cta[:,0].max()-t0)/1e3:.2f} us; exit min {ex[0]:.2f} p10 {ex[len(ex)//10]:.2f} med {np.median(ex):.2f} p90 {ex[9*len(ex)//10]:.2f} max {ex[-1]:.2f} us; units {cta[:,2].min()}-{cta[:,2].max()}")
t = full[:65536].reshape(-1, 16)
print("CTA0 unit | wg3 expander: before_go go_done sttm_issued st_done loop_end | issuer: before_sync synced issued  (clock64 cycles from CTA start)")
for k in range(30):
    print(k, *[f"{x:6d}" for x in t[k, :5]], "|", *[f"{x:6d}" for x in t[k, 8:11]])
