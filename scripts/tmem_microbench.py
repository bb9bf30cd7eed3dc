"""Run scripts/tmem_microbench.cu and print cycles per iteration for each mode."""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "tmem_microbench.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                "-o", so, os.path.join(HERE, "tmem_microbench.cu")], check=True)
lib = ctypes.CDLL(so)
lib.run_micro.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
iters = 4000
for mode, nbuf, grid, label in [
    (4, 1, 1, "MMA warp: wait(complete barrier) + 8 MMA N16 + commit"),
    (5, 1, 1, "MMA warp: 8 MMA N16 + commit, no wait"),
    (5, 2, 1, "MMA warp: 8 MMA N32 + commit, no wait"),
    (5, 3, 1, "MMA warp: 8 MMA N48 + commit, no wait"),
    (5, 4, 1, "MMA warp: 8 MMA N64 + commit, no wait"),
    (5, 8, 1, "MMA warp: 8 MMA N128 + commit, no wait"),
    (5, 16, 1, "MMA warp: 8 MMA N256 + commit, no wait"),
    (7, 2, 1, "e4m3 K32: 8 MMA N32 + commit"),
    (7, 3, 1, "e4m3 K32: 8 MMA N48 + commit"),
    (7, 4, 1, "e4m3 K32: 8 MMA N64 + commit"),
    (7, 8, 1, "e4m3 K32: 8 MMA N128 + commit"),
    (8, 2, 1, "i8 K32: 8 MMA N32 + commit"),
    (8, 4, 1, "i8 K32: 8 MMA N64 + commit"),
    (9, 1, 1, "f16 N16: commit every 4 groups"),
    (6, 1, 1, "SS: 8 MMA N16 + commit, no wait"),
    (6, 4, 1, "SS: 8 MMA N64 + commit, no wait"),
    (0, 0, 1, "STTM 4x16 cols + wait::st, 4 warps, 1 CTA"),
    (0, 0, 148, "STTM 4x16 cols + wait::st, 4 warps, 148 CTAs"),
    (1, 1, 1, "8 MMA (N16) + commit + wait round trip"),
    (2, 2, 1, "2 groups x 8 MMA in flight"),
    (2, 4, 1, "4 groups x 8 MMA in flight"),
    (2, 8, 1, "8 groups x 8 MMA in flight"),
    (3, 2, 1, "ping-pong STTM<->MMA, 2 buffers"),
    (3, 3, 1, "ping-pong STTM<->MMA, 3 buffers"),
    (3, 4, 1, "ping-pong STTM<->MMA, 4 buffers"),
    (3, 4, 148, "ping-pong STTM<->MMA, 4 buffers, 148 CTAs"),
]:
    out = np.zeros(grid * 2, np.int64)
    rc = lib.run_micro(mode, iters, nbuf, grid, out.ctypes.data)
    cyc = out.reshape(grid, 2).max(axis=1).mean() / iters
    extra = f" ({cyc / nbuf:.1f} per 8-MMA group)" if mode == 2 else ""
    print(f"mode {mode} nbuf {nbuf} grid {grid:3d}: {cyc:8.1f} cycles/iter{extra}   {label}  rc={rc}")
