"""Prefill-path debugging: repeatability and error vs the oracle for each kernel choice."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2410_23918_b200 as pkg
from oracle import bitstack_oracle as O
from synthetic import channel_gains, make_calibration, make_weight, make_x
from bitstack_test_helpers import stack_blocks

d_out, d_in, n = int(sys.argv[1]) if len(sys.argv) > 1 else 256, int(sys.argv[2]) if len(sys.argv) > 2 else 384, 4
g = channel_gains(d_in, 75); w = make_weight(d_out, d_in, 71)
s, blocks = O.compress(w, make_calibration(max(256, d_in), g, 72), n, 16, dtype="bf16")
s32 = s.astype(np.float32)
signs, u, v = stack_blocks(blocks, "bf16")
lay = pkg.Layer(d_out, d_in, 16, n, "bf16"); lay.load_blocks(0, signs, u, v, s32)
x = torch.from_numpy(make_x(40, g, 9).astype(np.float32)).cuda()
ref = O.matmul_dense(blocks, s32.astype(np.float64), n, x.cpu().numpy().astype(np.float64))
res = {}
for kern in ("auto", "prefill", "prefill", "tc", "simt", "auto"):
    lay.set_kernel(kern)
    y = lay.matmul(x); torch.cuda.synchronize()
    y = y.cpu().numpy().astype(np.float64)
    print(f"{kern:8s} rel {O.relative_l2(y, ref):.3e}", "same-as-prev-prefill" if kern in res and np.array_equal(res[kern], y) else "")
    res[kern] = y
d = np.abs(res["auto"] - res["prefill"])
print("auto vs prefill max diff", d.max(), "rows with diff", np.unique(np.nonzero(d > 1e-6)[1])[:20], "tokens", np.unique(np.nonzero(d > 1e-6)[0])[:20])
