"""Drive scripts/mma_selftest.cu: D = A B^T with A [128,16], B [16,16] (both K-major)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "mma_selftest.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler", "-fPIC",
                "-o", so, os.path.join(HERE, "mma_selftest.cu")], check=True)
lib = ctypes.CDLL(so)
lib.run_mma_test.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_uint, ctypes.c_int]
rng = np.random.default_rng(0)
A = rng.integers(-2, 3, (128, 16)).astype(np.float16)
Bm = rng.integers(-2, 3, (16, 16)).astype(np.float16)
ref = A.astype(np.float32) @ Bm.astype(np.float32).T
for mode in (0, 1):
    for swap in (0,):
        a = torch.from_numpy(A).cuda()
        b = torch.from_numpy(Bm).cuda()
        d = torch.full((128, 16), float("nan"), device="cuda")
        raw = torch.zeros((128, 16), dtype=torch.int32, device="cuda")
        rc = lib.run_mma_test(mode, a.data_ptr(), b.data_ptr(), d.data_ptr(), raw.data_ptr(), 0, swap)
        dd = d.cpu().numpy()
        ok = np.allclose(dd, ref)
        print(f"mode={'TS' if mode else 'SS'} swap={swap} rc={rc} ok={ok} nan={np.isnan(dd).sum()} "
              f"d[0,:4]={dd[0, :4]} ref[0,:4]={ref[0, :4]}")
        if mode == 1 and swap == 0:
            r = raw.cpu().numpy().view(np.uint32)[0, :8]
            print("   A in TMEM row0 cols 0..7:", [hex(int(x)) for x in r])
        if not ok and not np.isnan(dd).any():
            # try to identify a permutation: maybe D is A B^T with B transposed etc.
            for name, cand in (("A B", A.astype(np.float32) @ Bm.astype(np.float32)),):
                print("   matches", name, np.allclose(dd, cand))
sys.stdout.flush()
