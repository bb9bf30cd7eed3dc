"""Row-sharded TP ("distributed across multiple devices") with the
REAL library on GPUs: TPLayer + bitstack.Layer row shards + the all-gather, against the
unsharded oracle.

- world 2 over NCCL, one GPU per rank (skipped with fewer than 2 GPUs);
- world 2 over gloo with both ranks' shards on cuda:0 (the host-staged gather of tp.py): the
  composition TPLayer + Layer(row_begin, row_end) + gather on real kernels, runnable on the
  one-GPU boxes.  The ranks' kernels never wait on each other (the gather is host-side).

Each rank's y must be identical on every rank (the gather only moves bytes) and equal to the
oracle within the north-star bar (1e-3 relative L2 with bf16 factors)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, backend, d_out, d_in, n, results):
    import torch.distributed as dist
    from bitstack_test_helpers import stack_blocks
    from oracle import bitstack_oracle as O
    from synthetic import channel_gains, make_calibration, make_weight, make_x
    import paper_2410_23918_b200 as pkg
    from paper_2410_23918_b200.tp import TPLayer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    pkg.load_library()
    g = channel_gains(d_in, 31)
    w = make_weight(d_out, d_in, 30)
    s, blocks = O.compress(w, make_calibration(max(256, d_in), g, 32), n, 16, dtype="bf16", method="exact", seed=30)
    s32 = s.astype(np.float32)
    signs, u, v = stack_blocks(blocks, "bf16")
    lay = TPLayer(d_out, d_in, k=16, n_capacity=n, factor_dtype="bf16", device=dev)
    lay.load_blocks(0, signs, u, v, s32)
    out = {}
    for level in range(1, n + 1):
        lay.set_num_blocks(level)
        for batch in (1, 3, 24):               # MX decode (1 and 3 tokens) and the prefill GEMM
            x = make_x(batch, g, 40 + batch)
            xt = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).cuda()
            y = lay.matmul(xt)
            torch.cuda.synchronize()
            yn = y.double().cpu().numpy()
            ref = O.matmul_dense(blocks, s32.astype(np.float64), level, xt.double().cpu().numpy())
            # every rank holds the same bytes
            ys = [torch.zeros_like(y) for _ in range(world)]
            if backend == "nccl":
                dist.all_gather(ys, y)
            else:
                yc = y.cpu()
                ysc = [torch.zeros_like(yc) for _ in range(world)]
                dist.all_gather(ysc, yc)
                ys = ysc
            same = all(torch.equal(ys[0].cpu(), t.cpu()) for t in ys)
            out[(level, batch)] = (O.relative_l2(yn, ref), same, tuple(y.shape))
    results[rank] = out
    dist.destroy_process_group()


def _run(world, backend, d_out, d_in, n):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), backend, d_out, d_in, n, results), nprocs=world, join=True)
    for rank in range(world):
        for (level, batch), (err, same, shape) in results[rank].items():
            assert shape == (batch, d_out)
            assert same, (rank, level, batch)
            assert err <= 1e-3, (rank, level, batch, err)


@pytest.fixture(scope="module")
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_23918_b200 import build
    build.build()


@pytest.mark.parametrize("d_out", [512, 520])        # even shards, and shards of 260 rows
def test_tp_world2_gloo_real_library_one_gpu(built, d_out):
    _run(2, "gloo", d_out, 384, 3)


@pytest.mark.parametrize("d_out", [512, 520])
def test_tp_world2_nccl(built, d_out):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, "nccl", d_out, 384, 3)
