#!/usr/bin/env python
"""BitStack W_hat_n x on B200: us/layer and HBM GB/s vs peak (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload c2|c5]

One step = one bitstack_matmul of the workload's layer (the whole hot path: the
fused tcgen05 decode kernel; at N > 1 each rank computes its row shard and the
output slices are all-gathered over NCCL).  Blocks are synthetic stored-form
blocks from synthetic/ (kernel time does not depend on values); L2 is defeated
by rotating over enough layer copies that the working set exceeds 4x L2.
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (oracle/)
on the host cores on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import (CONFIGS, LLAMA31_8B_SHAPES, channel_gains,  # noqa: E402
                       make_random_blocks, make_x, seed_for)

L2_BYTES = 126 * 2 ** 20
WORKLOADS = {
    "c2": dict(CONFIGS["c2"], kind="decode",
               label="c2: Llama-3.1-8B q_proj 4096x4096, n=16 blocks, k=16, bf16 factors, decode"),
    "c5": dict(CONFIGS["c5"], kind="decode",
               label="c5: Llama-3.1-70B down_proj 8192x28672, n=12 blocks, k=16, bf16 factors, decode"),
    "c3_up": dict(CONFIGS["c3_up"], kind="prefill",
                  label="c3: Llama-3.1-8B up/gate_proj 14336x4096, n=8 blocks, k=16, bf16 factors, prefill 2048 tokens"),
    "c4": dict(d_out=4096, d_in=4096, n=4, k=16, batch=1, factor_dtype="bf16", kind="stack",
               label="c4: full Llama-3.1-8B linear stack (32 layers x q,k,v,o,gate,up,down = 224 matrices), "
                     "5541 MiB budget (levels from the budget with the Average ordering: 3-4 blocks per matrix, 3.88 in model-size units), "
                     "decode, one token-step = the 224 matmuls as 128 grouped calls (bitstack_matmul_grouped per shared input)"),
    "load": dict(CONFIGS["c5"], kind="load",
                 label="block streaming: the 12 blocks of Llama-3.1-70B down_proj 8192x28672 (k=16, bf16 "
                       "factors) pushed from pinned host memory with bitstack_load_blocks_async"),
    "compress": dict(CONFIGS["c2"], kind="compress",
                     label="GPU compression (Alg.1): Llama-3.1-8B q_proj 4096x4096, p=4096 calibration rows, "
                           "n=16 blocks, k=16, bf16 factors, randomized SVD (ell=32, 4 power iterations)"),
    "c3_down": dict(CONFIGS["c3_down"], kind="prefill",
                    label="c3: Llama-3.1-8B down_proj 4096x14336, n=8 blocks, k=16, bf16 factors, prefill 2048 tokens"),
}


def traffic_key(key):
    """DRAM read + write bytes of the roofline kernel(s) per launch (per token-step for C4) from
    profiles/traffic.json (one ncu capture, scripts/gpu_traffic.sh / gpu_c4_traffic.sh), or None."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(tpath) as f:
            return json.load(f).get(key)
    except Exception:  # noqa: BLE001
        return None


def peaks(kind="decode"):
    """Roofline denominator: HBM copy GB/s (decode), or dense bf16 TFLOP/s sustained (prefill
    GEMM with fp16 operands: same tensor rate as bf16, nominal ratio 1)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    key = "hbm_gbs" if kind == "decode" else "bf16_tflops_sustained"
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d[key]), f"measured (MEASURED_PEAKS.json {key})"
    except Exception:
        return (6650.0, "fallback (B200_PROFILING.md)") if kind == "decode" else \
            (2250.0, "fallback (nominal dense fp16/bf16)")


def alg_flops(w, rows, batch, n):
    """SURVEY §8(d) prefill: 2 r d_in (B + n k) (restore the tile on tensor cores + GEMM)."""
    return 2.0 * rows * w["d_in"] * (batch + n * w["k"])


def step_units(w, rows, batch, n):
    """The metric's numerator per step: GB (decode) or TFLOP (prefill)."""
    if w["kind"] == "decode":
        return alg_bytes_per_rank(w, rows, batch, n) / 1e9
    return alg_flops(w, rows, batch, n) / 1e12


def alg_bytes_per_rank(w, rows, batch, n, x_bytes=2, y_bytes=4):
    """n (r d_in / 8 + k (r + d_in) f) + B d_in |x| + B r |y| + 4 d_in."""
    return n * (rows * w["d_in"] / 8 + w["k"] * (rows + w["d_in"]) * 2) + batch * w["d_in"] * x_bytes \
        + batch * rows * y_bytes + 4 * w["d_in"]


class ClockSampler:
    """Polls NVML (SM clock, max clock, throttle reasons) every ~2 ms while active."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": names, "samples": len(self.samples)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def oracle_sample_time(w, n, batch, rows_sample, steps, warmup, seed):
    """Time the dense oracle (Eq.8 + Eq.4, fp64) for `rows_sample` output rows of the
    workload's layer: returns (seconds per step, algorithmic bytes per step)."""
    from oracle import bitstack_oracle as O
    d_out, d_in, k = w["d_out"], w["d_in"], w["k"]
    signs, u, v, s = make_random_blocks(n, d_out, d_in, k, seed=seed)
    u = O.round_to_dtype(u, "bf16")
    v = O.round_to_dtype(v, "bf16")
    rows = np.arange(rows_sample)
    sub = []
    for i in range(n):  # stored blocks restricted to the sampled rows (setup, untimed)
        sm = O.unpack_signs(signs[i], d_out, d_in)[rows]
        sub.append(O.Block(signs=O.pack_signs(sm), u=u[i][rows], v=v[i]))
    x = make_x(batch, channel_gains(d_in, seed + 1), seed + 2)
    for _ in range(warmup):
        O.matmul_dense(sub, s.astype(np.float64), n, x)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.matmul_dense(sub, s.astype(np.float64), n, x)
    dt = (time.perf_counter() - t0) / steps
    return dt, step_units(w, rows_sample, batch, n)


def metric_name(w):
    if w["kind"] == "decode":
        return "bitstack_matmul HBM GB/s (algorithmic bytes / time) [us/layer in ms_per_step]"
    return "bitstack_matmul prefill TFLOP/s (algorithmic 2 r d_in (B + n k) / time) [us/layer in ms_per_step]"


def unit_name(w):
    return "GB/s" if w["kind"] == "decode" else "TFLOP/s"



def run_stack(args, w, world, rank, local_rank):
    """Config C4: every linear of Llama-3.1-8B held as BitStack blocks at the
    paper's 5541 MiB memory point; one step = one decode token through all 224 matmuls
    (32 layers x 7), captured as one CUDA graph.  Row shards at N > 1 (outputs all-gathered)."""
    budget_mib = 5541
    names = list(LLAMA31_8B_SHAPES)
    # per-matrix levels from the memory budget with the Average ordering (budget.average_levels,
    # P:142-146): Eq.9 block sizes, 2004.5 MiB of embeddings / head / norms outside the stacks
    # (SURVEY Q15), a seeded permutation of the 224 matrices as the within-level order
    from paper_2410_23918_b200.budget import average_levels as budget_levels, prefix_levels, universal_stack
    eq9 = [(d_out * d_in + 16 * 16 * (d_out + d_in)) / 8.0
           for _ in range(32) for d_out, d_in in (LLAMA31_8B_SHAPES[nm] for nm in names)]
    order = np.random.default_rng(seed_for(4, 0, "blocks")).permutation(len(eq9)).tolist()
    if args.order == "random":   # the paper's Random sorting over n = 16 blocks per stack
        stack = universal_stack([16] * len(eq9), "random", seed=404)
        n_of = np.array(prefix_levels(stack, eq9, (budget_mib - 2004.5) * 2 ** 20)).reshape(32, len(names))
    else:
        n_of = np.array(budget_levels(eq9, (budget_mib - 2004.5) * 2 ** 20, order)).reshape(32, len(names))
    level = float(np.dot(n_of.reshape(-1), eq9) / sum(eq9))   # loaded levels in model-size units
    batch = args.batch or 1
    def oracle_stack_sample(reps):
        """The oracle on a bounded sample: 64 rows of each of layer 0's 7 matrices -> GB/s."""
        tot_bytes, tot_s = 0.0, 0.0
        for m, name in enumerate(names):
            d_out, d_in = LLAMA31_8B_SHAPES[name]
            ww = dict(d_out=d_out, d_in=d_in, k=16, kind="decode")
            nn = int(n_of[0, m])
            dt, _ = oracle_sample_time(ww, nn, batch, 64, reps, 1, seed_for(4, m, "blocks"))
            tot_bytes += step_units(ww, d_out, batch, nn) * 1e9     # the whole matrix ...
            tot_s += dt * d_out / 64                                # ... at the sampled per-row time
        return tot_bytes / 1e9 / tot_s, tot_s

    if args.impl == "reference":
        if rank != 0:
            return
        reps = max(1, min(args.steps // 100, 20))
        val, tot_s = oracle_stack_sample(reps)
        print(json.dumps({
            "impl": "reference", "metric": metric_name(dict(kind="decode")), "value": val, "unit": "GB/s",
            "n_gpus": world, "steps": reps, "warmup": 1, "ms_per_step": tot_s * 32 * 1e3,   # 32 layers per token
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (stored-form random blocks, synthetic/ recipe)",
            "config": {"workload": w["label"], "batch": batch, "parallelism": "cpu", "sample_rows": 64},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": "dense oracle (fp64 numpy) for 64 rows of each of layer 0's 7 matrices, "
                                       "scaled to whole matrices (x 32 layers for ms_per_step)"},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2410_23918_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    import paper_2410_23918_b200 as pkg
    pkg.load_library()
    # one set of stored-form blocks per matrix type (as many as the highest level), of which each
    # of the 32 handles loads its own level's prefix (every handle owns its device copy: 3.7 GB
    # of weights, the budget)
    layers, total_bytes = [], 0.0
    xs = {d: torch.from_numpy(make_x(batch, channel_gains(d, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
          for d in (4096, 14336)}
    for m, name in enumerate(names):
        d_out, d_in = LLAMA31_8B_SHAPES[name]
        nmax = max(1, int(n_of[:, m].max()))
        signs, u32, v32, s = make_random_blocks(nmax, d_out, d_in, 16, seed=seed_for(4, m, "blocks"))
        u_bf = torch.from_numpy(u32).to(torch.bfloat16)
        v_bf = torch.from_numpy(v32).to(torch.bfloat16)
        r0, r1 = d_out * rank // world, d_out * (rank + 1) // world
        for layer in range(32):
            nn = int(n_of[layer, m])
            lay = pkg.Layer(d_out, d_in, k=16, n_capacity=max(nn, 1), factor_dtype="bf16", row_begin=r0,
                            row_end=r1, device=local_rank)
            if nn:
                lay.load_blocks(0, signs[:nn], u_bf[:nn], v_bf[:nn], s)
            lay.set_num_blocks(nn)
            y = torch.empty((batch, r1 - r0), dtype=torch.float32, device="cuda")
            yf = torch.empty((world * batch, r1 - r0), dtype=torch.float32, device="cuda") if world > 1 else None
            layers.append((lay, xs[d_in], y, yf))
            total_bytes += alg_bytes_per_rank(dict(d_in=d_in, k=16), r1 - r0, batch, nn)
    stream = torch.cuda.current_stream()
    # matrices of one transformer layer that read the same activation run as one grouped call
    # (bitstack_matmul_grouped: one Zq + one decode launch): {q,k,v}, {o}, {gate,up}, {down}
    deps = [["q_proj", "k_proj", "v_proj"], ["o_proj"], ["gate_proj", "up_proj"], ["down_proj"]]
    if args.no_group:
        deps = [[nm] for nm in names]
    groups = []
    for layer in range(32):
        for dg in deps:
            mem = [layers[names.index(nm) * 32 + layer] for nm in dg]
            groups.append((pkg.Group([m[0] for m in mem], [m[1].data_ptr() for m in mem],
                                     [m[2].data_ptr() for m in mem]), mem))

    def token_step(sh):
        for grp, mem in groups:
            grp(pkg.BF16, pkg.F32, batch, sh)
            if world > 1:
                for _, _, y, yf in mem:
                    dist.all_gather_into_tensor(yf, y)

    for _ in range(max(args.warmup, 3)):
        token_step(stream.cuda_stream)
    torch.cuda.synchronize()
    l0 = pkg.launch_count()
    token_step(stream.cuda_stream)
    per_step_launches = pkg.launch_count() - l0
    steps = max(3, min(args.steps, 200))
    graph = None
    if world == 1 and not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            token_step(cap.cuda_stream)
        stream.wait_stream(cap)
        graph.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            if graph is not None:
                graph.replay()
            else:
                token_step(stream.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        pkg.profile_begin(4096)
        token_step(stream.cuda_stream)
        torch.cuda.synchronize()
        nk, kms = pkg.profile_end()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tb = torch.tensor([total_bytes], dtype=torch.float64, device="cuda")
        dist.all_reduce(tb)
        all_bytes = float(tb.item())
    else:
        all_bytes = total_bytes
    # e2e: the token's activations in from pinned host memory and every output back
    x_h = {d: x.cpu().pin_memory() for d, x in xs.items()}
    y_h = [torch.empty_like(y, device="cpu").pin_memory() for _, _, y, _ in layers]
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ke = max(3, min(steps, 50))
    f0.record()
    for _ in range(ke):
        for d, x in xs.items():
            x.copy_(x_h[d], non_blocking=True)
        if graph is not None:
            graph.replay()
        else:
            token_step(stream.cuda_stream)
        for (_, _, y, _), yh in zip(layers, y_h):
            yh.copy_(y, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / ke
    clocks = sampler.summary()
    peak, peak_src = peaks("decode")
    if graph is not None:   # the token's kernel pairs ARE the graph-replayed step
        nk, kms = per_step_launches * steps, ms
    achieved = total_bytes / 1e9 / (kms * 1e-3) if kms > 0 else None
    if rank == 0:
        line = {
            "metric": metric_name(dict(kind="decode")) + " -- whole 8B linear stack per token",
            "value": all_bytes / 1e9 / (ms * 1e-3), "unit": "GB/s", "n_gpus": world, "steps": steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "tokens_per_s": batch / (ms * 1e-3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "e4m3 MMA operands (S exact; Z as 3 e4m3 digits with per-32-channel UE8M0 scales), fp32 accumulate",
            "data": "synthetic (stored-form random blocks + activations, synthetic/ recipe)",
            "config": {"workload": w["label"], "batch": batch, "matrices": len(layers),
                       "blocks_per_matrix": {str(v): int((n_of == v).sum()) for v in sorted(set(n_of.reshape(-1).tolist()))},
                       "budget_mib": budget_mib, "loaded_level": level,
                       "weight_bytes_per_token": all_bytes,
                       "parallelism": f"tp{world} (row shards + NCCL all-gather)" if world > 1 else "tp1",
                       "l2": "inputs larger than L2 (3.7 GB of blocks per token-step)",
                       "calls_per_token": len(groups),
                       "grouping": "per matrix" if args.no_group else "grouped per shared input: {q,k,v},{o},{gate,up},{down}",
                       "sorting": args.order, "level_range": [int(n_of.min()), int(n_of.max())],
                       "timing": "CUDA-graph replay of the token's calls" if graph is not None else "eager launches"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": (None if args.no_group or args.order != "average"
                                     else traffic_key(f"c4_b{batch}_g{world}")),
                         "peak_source": peak_src,
                         "kernel": "zq_mx + decode_mx kernel pairs (all of the token's calls: the graph-replayed step)",
                         "kernel_us": kms * 1e3, "kernel_launches_timed": nk},
            "clocks": clocks,
            "e2e": {"value": all_bytes / 1e9 / (e2e_ms * 1e-3), "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in x_h.values())),
                    "d2h_bytes_per_step": int(sum(y.numel() * y.element_size() for y in y_h))},
            "gpu_launches": int(per_step_launches * steps),
            "cpu_baseline": None,
        }
        if world == 1 and not args.no_cpu_baseline:
            v, _ = oracle_stack_sample(1)
            line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
                                    "sample": "dense oracle (fp64 numpy, Eq.8+Eq.4) for 64 rows of each of "
                                              "layer 0's 7 matrices, 1 call each"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_load(args, w, world, rank, local_rank):
    """Block streaming (Fig.2 "load more weight residuals from
    storage when available memory increases"): one step = pushing all n blocks of the
    workload's matrix from pinned host memory into a handle with bitstack_load_blocks_async
    (DMA of this rank's row shard of S_i and U_i plus V_i into staging, on-device repack into
    the tile layout), timed with CUDA events on the load stream.  Reported beside it: a plain
    pinned cudaMemcpyAsync of the same bytes (the PCIe roofline) and the load overlapped with
    back-to-back decode calls of a resident copy of the same matrix on another stream."""
    d_out, d_in, k, n = w["d_out"], w["d_in"], w["k"], args.n or w["n"]
    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import bitstack_oracle as O
        signs, _, _, _ = make_random_blocks(1, d_out, d_in, k, seed=seed_for(5, 0, "blocks"))
        reps = max(1, min(args.steps, 3))
        O.unpack_signs(signs[0], d_out, d_in)
        t0 = time.perf_counter()
        for _ in range(reps):
            O.unpack_signs(signs[0], d_out, d_in)
        dt = (time.perf_counter() - t0) / reps
        val = signs[0].nbytes / 1e9 / dt
        print(json.dumps({
            "impl": "reference", "metric": "block load GB/s (stored-form bytes made usable per second)", "value": val,
            "unit": "GB/s", "n_gpus": world, "steps": reps, "warmup": 1, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (random stored-form blocks)",
            "config": {"workload": w["label"], "parallelism": "cpu"},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": "oracle unpack_signs (canonical bits -> +-1) of one block"},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2410_23918_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    import paper_2410_23918_b200 as pkg
    pkg.load_library()
    signs, u32, v32, s = make_random_blocks(n, d_out, d_in, k, seed=seed_for(5, 0, "blocks"))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    ps = pin(signs)
    pu = torch.from_numpy(u32).to(torch.bfloat16).pin_memory()
    pv = torch.from_numpy(v32).to(torch.bfloat16).pin_memory()
    pss = pin(s)
    r0, r1 = d_out * rank // world, d_out * (rank + 1) // world
    rows = r1 - r0
    step_bytes = n * (rows * d_in / 8 + k * (rows + d_in) * 2) + 4 * d_in
    lay = pkg.Layer(d_out, d_in, k=k, n_capacity=n, factor_dtype="bf16", row_begin=r0, row_end=r1, device=local_rank)
    busy = pkg.Layer(d_out, d_in, k=k, n_capacity=n, factor_dtype="bf16", row_begin=r0, row_end=r1, device=local_rank)
    busy.load_blocks(0, ps, pu, pv, pss)
    side = torch.cuda.Stream()
    l0 = pkg.launch_count()

    def load_step():
        lay.load_blocks_async(0, ps, pu, pv, pss, stream=side)

    for _ in range(args.warmup):
        load_step()
    torch.cuda.synchronize()
    launches_per_step = (pkg.launch_count() - l0) // args.warmup
    steps = max(3, min(args.steps, 20))
    sampler = ClockSampler(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(side)
        for _ in range(steps):
            load_step()
        e1.record(side)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # PCIe roofline: plain pinned host->device copies of the same pinned sign buffer the load
    # reads (best of 10), scaled to the step's bytes
    dflat = torch.empty(ps.numel(), dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(10):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        dflat.copy_(ps.view(-1), non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        best = min(best, c0.elapsed_time(c1))
    pcie_gbs = ps.numel() / 1e9 / (best * 1e-3)
    del dflat
    # overlap: decode of the resident copy on the main stream while the load runs on `side`
    x = torch.from_numpy(make_x(1, channel_gains(d_in, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
    y = torch.empty((1, rows), dtype=torch.float32, device="cuda")
    main = torch.cuda.current_stream()
    calls = 40
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        busy.matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, 1, main.cuda_stream)
    torch.cuda.synchronize()
    d0.record(main)
    for _ in range(calls):
        busy.matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, 1, main.cuda_stream)
    d1.record(main)
    torch.cuda.synchronize()
    dec_alone = d0.elapsed_time(d1) / calls
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(main)
    g0.record(side)
    load_step()
    g1.record(side)
    ov_calls = 0
    while not g1.query() or ov_calls < 5:
        busy.matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, 1, main.cuda_stream)
        ov_calls += 1
        if ov_calls % 20 == 0:
            main.synchronize()
        if ov_calls > 20000:
            break
    d1.record(main)
    torch.cuda.synchronize()
    ov_load_ms = g0.elapsed_time(g1)
    dec_ov = d0.elapsed_time(d1) / ov_calls
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_bytes = step_bytes * world
    if rank == 0:
        peak_src = "measured in-run: pinned host->device cudaMemcpyAsync of the pinned sign buffer (best of 10)"
        line = {
            "metric": "block load GB/s (stored-form bytes of the rank's shard moved from pinned host memory into the "
                      "device block store per second)",
            "value": total_bytes / 1e9 / (ms * 1e-3), "unit": "GB/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_block": ms / n, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8 signs + bf16 factors",
            "data": "synthetic (random stored-form blocks in pinned host memory)",
            "config": {"workload": w["label"], "d_out": d_out, "d_in": d_in, "n": n, "k": k,
                       "bytes_per_step": total_bytes, "parallelism": f"tp{world} (row shards)" if world > 1 else "tp1",
                       "l2": "inputs larger than L2 (host memory, 355 MB per step)"},
            "roofline": {"bound": "pcie", "achieved": step_bytes / 1e9 / (ms * 1e-3), "peak": pcie_gbs, "unit": "GB/s",
                         "frac": (step_bytes / 1e9 / (ms * 1e-3)) / pcie_gbs, "traffic": None, "peak_source": peak_src,
                         "kernel": "cudaMemcpyAsync DMA (overlapped) + repack_rows_kernel + factor_max_kernel + factor_scale_kernel per block"},
            "overlap": {"decode_us_alone": dec_alone * 1e3, "decode_us_during_load": dec_ov * 1e3,
                        "decode_calls_during_load": ov_calls, "load_ms_during_decode": ov_load_ms,
                        "load_gbs_during_decode": step_bytes / 1e9 / (ov_load_ms * 1e-3)},
            "clocks": sampler.summary(),
            "e2e": {"value": total_bytes / 1e9 / (ms * 1e-3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(step_bytes), "d2h_bytes_per_step": 0,
                    "note": "the step itself is the host->device transfer"},
            "gpu_launches": int(launches_per_step * steps),
            "cpu_baseline": None,
        }
        if world == 1 and not args.no_cpu_baseline:
            from oracle import bitstack_oracle as O
            O.unpack_signs(signs[0], d_out, d_in)
            t0 = time.perf_counter()
            O.unpack_signs(signs[0], d_out, d_in)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": signs[0].nbytes / 1e9 / dt, "unit": "GB/s", "cores": cpu_cores(),
                                    "kind": "oracle", "sample": "oracle unpack_signs of one block (canonical bits -> +-1)"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def compress_flops(d_out, d_in, k, ell=32, q=4):
    """Algorithmic flops of one block of bitstack_compress: the 2q + 2 skinny GEMMs with |R|
    (2 d_out d_in ell each), the left-vector GEMM and the residual update (2 k d_out d_in)."""
    return (2 * q + 2) * 2.0 * d_out * d_in * ell + 2.0 * d_out * ell * k + 2.0 * k * d_out * d_in


def run_compress(args, w, world, rank, local_rank):
    """Alg.1 for one matrix on the GPU (bitstack_compress).  One step =
    compressing the workload's matrix into n blocks from W and the calibration activations
    already in device memory; the metric is algorithmic TFLOP/s (compress_flops) against the
    FP32 CUDA-core peak (the GEMMs run as cuBLAS SGEMM without TF32).  Replicas only at N > 1
    (each rank compresses its own copy; there is no exchange step)."""
    d_out, d_in, k, n = w["d_out"], w["d_in"], w["k"], args.n or w["n"]
    p_cal = 4096
    step_flops = n * compress_flops(d_out, d_in, k)

    def oracle_sample():
        from oracle import bitstack_oracle as O
        dd = 1024
        g = channel_gains(dd, 9)
        ww = np.random.default_rng(1).standard_normal((dd, dd)) * 0.02
        xc = np.random.default_rng(2).standard_normal((1024, dd)) * g[None, :]
        t0 = time.perf_counter()
        O.compress(ww, xc, 1, k, dtype="bf16", method="randomized")
        dt = time.perf_counter() - t0
        return compress_flops(dd, dd, k) / dt / 1e12, dt

    if args.impl == "reference":
        if rank != 0:
            return
        val, dt = oracle_sample()
        print(json.dumps({
            "impl": "reference", "metric": "bitstack_compress TFLOP/s (algorithmic)", "value": val, "unit": "TFLOP/s",
            "n_gpus": world, "steps": 1, "warmup": 0, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w["label"], "parallelism": "cpu"},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": "oracle compress (randomized SVD, fp64 numpy) of one 1024x1024 block"},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2410_23918_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    import paper_2410_23918_b200 as pkg
    pkg.load_library()
    from synthetic import make_calibration, make_weight
    g = channel_gains(d_in, 5)
    wt = torch.from_numpy(make_weight(d_out, d_in, 3).astype(np.float32)).cuda()
    xt = torch.from_numpy(make_calibration(p_cal, g, 4).astype(np.float32)).cuda()
    for _ in range(max(1, min(args.warmup, 3))):
        pkg.compress(wt, xt, n, k)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 5))
    l0 = pkg.launch_count()
    sampler = ClockSampler(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            out = pkg.compress(wt, xt, n, k)
        e1.record()
        torch.cuda.synchronize()
    launches = pkg.launch_count() - l0
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # e2e: W and X_cal from pinned host memory, the stored form back to pinned host memory
    wh, xh = wt.cpu().pin_memory(), xt.cpu().pin_memory()
    outs_h = [o.cpu().pin_memory() for o in out[:4]]
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    wd, xd = wh.cuda(non_blocking=True), xh.cuda(non_blocking=True)
    res = pkg.compress(wd, xd, n, k)
    for o, oh in zip(res[:4], outs_h):
        oh.copy_(o, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    resid = out[5].cpu().numpy()
    peak = 148 * 128 * 2 * 1.965e9 / 1e12
    if rank == 0:
        line = {
            "metric": "bitstack_compress TFLOP/s (algorithmic: skinny GEMMs with |R| + residual update)",
            "value": world * step_flops / 1e12 / (ms * 1e-3), "unit": "TFLOP/s", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_block": ms / n, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (GEMMs, QR, SVD), bf16 stored factors",
            "data": "synthetic (W ~ N(0, 0.02^2), calibration activations with outlier channels)",
            "config": {"workload": w["label"], "d_out": d_out, "d_in": d_in, "n": n, "k": k, "p": p_cal,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "working set 3 x 64 MiB fp32 matrices per block pass (> L2)",
                       "residual_norms": [float(x) for x in resid]},
            "roofline": {"bound": "alu", "achieved": step_flops / 1e12 / (ms * 1e-3), "peak": peak, "unit": "TFLOP/s",
                         "frac": step_flops / 1e12 / (ms * 1e-3) / peak, "traffic": None,
                         "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (B200_PROFILING.md unit counts)",
                         "kernel": "whole compression step (cuBLAS SGEMM dominates)"},
            "clocks": sampler.summary(),
            "e2e": {"value": world * step_flops / 1e12 / (e2e_ms * 1e-3), "unit": "TFLOP/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(wh.numel() * 4 + xh.numel() * 4),
                    "d2h_bytes_per_step": int(sum(o.numel() * o.element_size() for o in outs_h))},
            "gpu_launches": int(launches),
            "cpu_baseline": None,
        }
        if world == 1 and not args.no_cpu_baseline:
            val, dt = oracle_sample()
            line["cpu_baseline"] = {"value": val, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle",
                                    "sample": "oracle compress (randomized SVD, fp64 numpy) of one 1024x1024 block"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def relaunch(n):
    """`--gpus N` without a launcher: run N ranks of this command under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and pass rank 0's line through."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    sys.stdout.write(proc.stdout)
    if proc.returncode != 0:
        sys.exit(proc.returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--n", type=int, default=None, help="active blocks (default: the config's n)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replay")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-group", action="store_true",
                    help="c4: one bitstack_matmul per matrix instead of grouped calls per shared input")
    ap.add_argument("--order", choices=["average", "random"], default="average",
                    help="c4: the universal stack's sorting (P:351); Greedy needs measured perplexities")
    ap.add_argument("--sweep", action="store_true", help="also report us/layer for n = 1, 2, 4, 8, 16")
    ap.add_argument("--kernel", choices=["auto", "tc", "prefill", "rgemv", "simt"], default="auto",
                    help="decode workloads: force one path (bitstack_set_kernel) for crossover sweeps")
    ap.add_argument("--shard", type=int, default=1,
                    help="decode, one GPU: time rank 0's row shard of a G-way row split (the per-rank "
                         "kernel of SURVEY §8(e) at r_G = d_out / G rows, V and s replicated)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    w = dict(WORKLOADS[args.workload])
    n = args.n or w["n"]
    batch = args.batch or w["batch"]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if w["kind"] == "stack":
        return run_stack(args, w, world, rank, local_rank)
    if w["kind"] == "load":
        return run_load(args, w, world, rank, local_rank)
    if w["kind"] == "compress":
        return run_compress(args, w, world, rank, local_rank)

    if args.impl == "reference":
        if rank != 0:
            return
        budget_s = 60.0
        # bounded row sample: calibrate on 16 rows, then size the per-step sample (>= 1 row) so
        # that --steps K --warmup W fit the budget; with a very large K only as many steps as
        # fit are timed (reported in "steps")
        t16, _ = oracle_sample_time(w, n, batch, 16, 1, 0, seed_for(2, 0, "blocks"))
        t_row = max(t16 / 16.0, 1e-7)
        rows = int(max(16, min(w["d_out"], budget_s / (t_row * (args.steps + args.warmup)))))
        steps_run = int(min(args.steps, max(3, budget_s / (t_row * rows))))
        warm_run = min(args.warmup, 3)
        dt, _ = oracle_sample_time(w, n, batch, rows, steps_run, warm_run, seed_for(2, 0, "blocks"))
        # the whole layer's work at the sampled per-row time (the per-block V / x terms of a
        # row sample would otherwise inflate a small sample's throughput)
        val = step_units(w, w["d_out"], batch, n) / (dt * w["d_out"] / rows)
        line = {
            "impl": "reference", "metric": metric_name(w), "value": val, "unit": unit_name(w), "n_gpus": world, "steps": steps_run, "warmup": warm_run,
            "ms_per_step": dt * 1e3 * w["d_out"] / rows, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (stored-form random blocks, synthetic/ recipe)",
            "config": {"workload": w["label"], "d_out": w["d_out"], "d_in": w["d_in"], "n": n, "k": w["k"],
                       "batch": batch, "parallelism": "cpu", "sample_rows": rows,
                       "timing": "per-step row sample, scaled to the whole layer"},
            "cpu_baseline": {"value": val, "unit": unit_name(w), "cores": cpu_cores(), "kind": "oracle",
                             "sample": f"dense oracle (fp64 numpy) for {rows} of {w['d_out']} output rows, all {n} blocks"},
            "e2e": {"value": val, "unit": unit_name(w), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2410_23918_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    import paper_2410_23918_b200 as pkg
    pkg.load_library()

    d_out, d_in, k = w["d_out"], w["d_in"], w["k"]
    if args.shard > 1:
        assert world == 1, "--shard G times one rank's shard on one GPU"
        r0, r1 = 0, d_out // args.shard
    else:
        r0 = d_out * rank // world
        r1 = d_out * (rank + 1) // world
    rows = r1 - r0
    # ---- layer copies: working set per rank >= 4 x L2 (inputs larger than L2)
    per_layer = alg_bytes_per_rank(w, rows, batch, n)
    copies = max(2, math.ceil(4 * L2_BYTES / per_layer))
    signs, u32, v32, s = make_random_blocks(w["n"], d_out, d_in, k, seed=seed_for(2, 0, "blocks"))
    u_bf = torch.from_numpy(u32).to(torch.bfloat16)
    v_bf = torch.from_numpy(v32).to(torch.bfloat16)
    layers = []
    for c in range(copies):
        lay = pkg.Layer(d_out, d_in, k=k, n_capacity=w["n"], factor_dtype="bf16", row_begin=r0, row_end=r1,
                        device=local_rank)
        lay.load_blocks(0, signs, u_bf, v_bf, s)
        lay.set_num_blocks(n)
        if args.kernel != "auto":
            lay.set_kernel(args.kernel)
        layers.append(lay)
    x = torch.from_numpy(make_x(batch, channel_gains(d_in, 5), 6).astype(np.float32)).to(torch.bfloat16).cuda()
    y = torch.empty((batch, rows), dtype=torch.float32, device="cuda")
    y_full = torch.empty((world, batch, rows), dtype=torch.float32, device="cuda") if world > 1 else None
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    def step(i):
        layers[i % copies].matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, batch, sh)
        if world > 1:
            dist.all_gather_into_tensor(y_full, y)

    def timed(nsteps, use_graph):
        """Device time of `nsteps` steps: CUDA-graph replays (the graph is captured, then
        replayed once untimed so that its upload is not in the number), or eager launches."""
        graph = None
        if use_graph:
            gs = min(nsteps, copies * max(1, 256 // copies))
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(graph, stream=cap):
                for i in range(gs):
                    layers[i % copies].matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, batch,
                                                  cap.cuda_stream)
            stream.wait_stream(cap)
            graph.replay()               # untimed: graph upload / first-launch costs
            reps = max(1, nsteps // gs)
            nsteps = reps * gs
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = pkg.launch_count()
        e0.record()
        if graph is not None:
            for _ in range(reps):
                graph.replay()
        else:
            for i in range(nsteps):
                step(i)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        launches = pkg.launch_count() - l0 if graph is None else nsteps * per_step_launches
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, nsteps, launches

    use_graph = (not args.no_graph) and world == 1
    # warm-up: at least one call per layer copy, so every copy's lazily sized workspaces exist
    # before any CUDA-graph capture (a workspace allocation cannot happen while capturing)
    for i in range(max(args.warmup, copies)):
        step(i)
    torch.cuda.synchronize()
    l0 = pkg.launch_count()
    step(0)
    per_step_launches = pkg.launch_count() - l0   # our kernels per bitstack_matmul call
    torch.cuda.synchronize()
    # bitstack_matmul AUTO with bf16 factors (csrc/bitstack.cu choose_path): the e4m3 decode up to
    # 5 tokens, restore-and-multiply for 6..32, the prefill GEMM above (shards of >= 128 rows)
    if args.kernel == "auto":
        path = "decode" if (batch <= 5 or rows < 128) else ("rgemv" if batch <= 32 else "prefill")
    else:
        path = {"tc": "decode", "simt": "decode"}.get(args.kernel, args.kernel)
    decode_path = path == "decode"

    sampler = ClockSampler(local_rank)
    with sampler:
        ms, ksteps, launches = timed(args.steps, use_graph)
        if decode_path and use_graph:
            # the dominant kernel is the step: the zq + decode pair (one PDL pair per <= 8 tokens)
            # is all a decode step launches, so its per-launch time is the graph-replayed step
            nk, kms = ksteps, ms
        else:
            # prefill: the GEMM alone, bracketed by CUDA events on its stream (eager launches of
            # ~0.2 ms kernels: launch gaps are negligible); N > 1: the decode pair without the
            # collective
            kp = min(max(args.steps, 16), 256)
            pkg.profile_begin(kp)
            for i in range(kp):
                layers[i % copies].matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, batch, sh)
            torch.cuda.synchronize()
            nk, kms = pkg.profile_end()
    clocks = sampler.summary()
    ms_step = ms / ksteps
    total_units = step_units(w, rows, batch, n)  # this rank
    if world > 1:
        tb = torch.tensor([total_units], dtype=torch.float64, device="cuda")
        dist.all_reduce(tb)
        total_units = float(tb.item())
    value = total_units / (ms_step * 1e-3)
    kernel_ms = kms / max(nk, 1)
    assert kernel_ms <= ms_step * (1.02 if use_graph and decode_path else 1.1) or world > 1, (kernel_ms, ms_step)   # a kernel cannot outlast its step
    if decode_path:   # dominant kernel: the zq + decode PDL pair(s), algorithmic bytes
        dom_units = alg_bytes_per_rank(w, rows, batch, n) / 1e9
        nbk = min(batch, 8)
        dom_name = "bs::zq_mx_kernel<%d> + bs::decode_mx_kernel<%d> (PDL pair%s)" % (
            nbk, nbk, "" if batch <= 8 else ", %d pairs per call" % ((batch + 7) // 8))
    elif path == "rgemv":   # dominant kernel: the restore; each product P_i[j, c] (fp32) is read once from TMEM
        dom_units = 4.0 * n * rows * d_in / 1e12   # TB of TMEM reads per launch
        dom_name = "bs::rgemv_kernel<%d> (restore-and-multiply)" % (16 if batch <= 16 else 32)
    else:             # dominant kernel: the GEMM, 2 B r d_in flops
        dom_units = 2.0 * batch * rows * d_in / 1e12
        dom_name = "bs::prefill_gemm_kernel<BN> (BN = 128 or 256 by wave fill)"
    achieved = dom_units / (kernel_ms * 1e-3)
    issue_frac = None
    if path == "rgemv":
        # TMEM-read roofline: tcgen05.ld moves 64 B per clock per SM (B300_MICROARCH.md "LDTM
        # throughput", the same TMEM design on sm_100a) at the max SM clock; the restore reads every
        # fp32 product once.  Also reported: the issue fraction (2.5 lane-instructions per element
        # and block against 128 per clock per SM).
        mhz = float((clocks or {}).get("sm_max_mhz") or 1965.0)
        sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
        peak, peak_src = sms * 64 * mhz * 1e6 / 1e12, "derived: SMs x 64 B/clk TMEM read x max SM clock (B300_MICROARCH.md LDTM throughput)"
        issue_frac = (2.5 * n * rows * d_in) / (kernel_ms * 1e-3) / (sms * 128 * mhz * 1e6)
    else:
        peak, peak_src = peaks("decode" if decode_path else "prefill")
    traffic = traffic_key(f"{args.workload}_n{n}_b{batch}_g{world}" + ("_rgemv" if path == "rgemv" else ""))

    # ---- e2e: public API with host buffers (pinned), copies inside the timed region
    x_h = x.cpu().pin_memory()
    y_h = torch.empty((batch, d_out if world > 1 else rows), dtype=torch.float32).pin_memory()
    ke = min(args.steps, 2000)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if use_graph:
        # the same public calls (H2D copy, bitstack_matmul, D2H copy) captured into a CUDA
        # graph, as a serving loop would issue them; every step still moves x in and y out
        gs = min(ke, copies * max(1, 64 // copies))
        for lay in layers:   # first host-buffer call of each layer outside capture (staging allocation)
            lay.matmul_raw(x_h.data_ptr(), pkg.BF16, y_h.data_ptr(), pkg.F32, batch, sh)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            for i in range(gs):   # host x in, host y out: bitstack_matmul moves them (C ABI host path)
                layers[i % copies].matmul_raw(x_h.data_ptr(), pkg.BF16, y_h.data_ptr(), pkg.F32, batch,
                                              cap.cuda_stream)
        stream.wait_stream(cap)
        reps = max(1, ke // gs)
        ke = reps * gs
        graph.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            graph.replay()
        e1.record()
    else:
        e0.record()
        for i in range(ke):
            x.copy_(x_h, non_blocking=True)
            layers[i % copies].matmul_raw(x.data_ptr(), pkg.BF16, y.data_ptr(), pkg.F32, batch, sh)
            if world > 1:
                dist.all_gather_into_tensor(y_full, y)
                y_h.copy_(y_full.permute(1, 0, 2).reshape(batch, d_out), non_blocking=True)
            else:
                y_h.copy_(y, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / ke
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": total_units / (e2e_ms * 1e-3), "unit": unit_name(w), "ms_per_step": e2e_ms,
           "timing": ("CUDA-graph replay of bitstack_matmul on pinned HOST x / y (the library moves them)"
                      if use_graph else "eager: H2D copy + bitstack_matmul + D2H copy"),
           "h2d_bytes_per_step": int(x_h.numel() * x_h.element_size()),
           "d2h_bytes_per_step": int(y_h.numel() * y_h.element_size())}

    sweep = None
    if args.sweep and world == 1 and w["kind"] == "decode":
        sweep = {}
        for nn in (1, 2, 4, 8, 16):
            if nn > w["n"]:
                continue
            for lay in layers:
                lay.set_num_blocks(nn)
            per = alg_bytes_per_rank(w, rows, batch, nn)
            cp = max(2, math.ceil(4 * L2_BYTES / per))
            cp = min(cp, copies)
            msn, kn, _ = timed(max(2000, 4 * cp), use_graph)
            us = msn / kn * 1e3
            sweep[str(nn)] = {"us_per_layer": us, "GBps": per / (us * 1e-6) / 1e9,
                              "l2_note": "rotation" if cp * per >= 4 * L2_BYTES else "partially L2-resident"}
        for lay in layers:
            lay.set_num_blocks(n)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.shard == 1:
        # bounded sample, ~10-15 s of CPU work: calibrate on 256 rows, then calls of ~3 s each
        dt0, _ = oracle_sample_time(w, n, batch, 256, 1, 0, seed_for(2, 0, "blocks"))
        rows_s = int(min(d_out, 256 * max(1, int(3.0 / max(dt0, 1e-3)))))
        steps_s = int(max(1, min(10, round(12.0 / max(dt0 * rows_s / 256, 1e-3)))))
        dt, _ = oracle_sample_time(w, n, batch, rows_s, steps_s, 0, seed_for(2, 0, "blocks"))
        cpu = {"value": step_units(w, d_out, batch, n) / (dt * d_out / rows_s), "unit": unit_name(w),
               "cores": cpu_cores(), "kind": "oracle",
               "sample": f"dense oracle (fp64 numpy, Eq.8+Eq.4) for {rows_s} of {d_out} output rows, "
                         f"all {n} blocks, {steps_s} calls ({dt * steps_s:.1f} s of CPU work), scaled to the whole layer"}

    # N > 1: the NCCL all-gather of the output slices timed alone (kernel,
    # collective and end-to-end reported separately); all ranks take part
    coll = None
    if world > 1:
        try:
            reps = 200
            dist.barrier()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for _ in range(reps):
                dist.all_gather_into_tensor(y_full, y)
            g1.record()
            torch.cuda.synchronize()
            t = torch.tensor([g0.elapsed_time(g1) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            coll = {"op": "NCCL all_gather_into_tensor of the fp32 y slices", "us": float(t.item()) * 1e3,
                    "bytes_per_rank": int(y.numel() * y.element_size())}
        except Exception as ex:  # noqa: BLE001 -- the main line must still print
            coll = {"error": str(ex)[:200]}
    if rank == 0:
        line = {
            "metric": metric_name(w),
            "value": value, "unit": unit_name(w), "n_gpus": world, "steps": ksteps, "warmup": args.warmup,
            "ms_per_step": ms_step, "us_per_layer": ms_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": ("e4m3 MMA operands (S exact; Z as 3 e4m3 digits with per-32-channel UE8M0 scales), fp32 accumulate" if w["kind"] == "decode"
                      else "bf16 restore MMA + fp16 GEMM operands, fp32 accumulate"),
            "data": "synthetic (stored-form random blocks + activations, synthetic/ recipe)",
            "config": {"workload": w["label"], "d_out": d_out, "d_in": d_in, "n": n, "k": k, "batch": batch,
                       "factor_dtype": "bf16", "x_dtype": "bf16", "y_dtype": "f32",
                       "parallelism": f"tp{world} (row shards + NCCL all-gather)" if world > 1 else "tp1",
                       "l2": f"inputs larger than L2: rotation over {copies} layer copies "
                             f"({copies * per_layer / 2 ** 20:.0f} MiB/rank > 4x126 MiB)",
                       "timing": "CUDA-graph replay" if use_graph else "eager launches"},
            "roofline": {"bound": {"decode": "hbm", "rgemv": "tmem", "prefill": "tensor"}[path], "achieved": achieved,
                         "peak": peak, "unit": {"decode": "GB/s", "rgemv": "TB/s", "prefill": "TFLOP/s"}[path],
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": dom_name, "kernel_us": kernel_ms * 1e3,
                         "kernel_launches_timed": nk,
                         {"decode": "bytes_per_launch", "rgemv": "tmem_bytes_per_launch", "prefill": "flops_per_launch"}[path]:
                             dom_units * (1e9 if decode_path else 1e12)},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
        }
        if issue_frac is not None:
            line["roofline"]["issue_frac"] = issue_frac
        if args.shard > 1:
            line["config"]["parallelism"] = f"rank 0 of a tp{args.shard} row split, timed alone on one GPU"
            line["config"]["shard"] = {"of": args.shard, "rows": rows,
                                       "hbm_floor_us": dom_units * 1e9 / (peak * 1e9) * 1e6,
                                       "note": "value = this rank's units / its step time (no collective)"}
        if sweep:
            line["n_sweep"] = sweep
        if coll is not None:
            line["collective"] = coll
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
