"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded TP host logic.

Each rank computes its row shard's y with the oracle (a stand-in for the CUDA library,
which needs a GPU) and the shared gather/reorder code assembles y; the result must equal
the unsharded oracle y exactly (the gather only moves bytes)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bitstack_oracle as O
from paper_2410_23918_b200.tp import TPLayer, gather_rows, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleShard:
    """Stand-in for bitstack.Layer on CPU: stores its row shard, computes y with the oracle."""

    def __init__(self, d_out, d_in, k=16, n_capacity=16, factor_dtype="f32", row_begin=0, row_end=None,
                 device=None):
        self.d_out, self.d_in, self.r0, self.r1 = d_out, d_in, row_begin, row_end
        self.blocks, self.s, self.n = [], None, 0

    def load_blocks(self, first_block, signs, u, v, s=None, stream=None):
        if s is not None:
            self.s = np.asarray(s, np.float64)
        del self.blocks[first_block:]
        for i in range(signs.shape[0]):
            sm = O.unpack_signs(signs[i], self.d_out, self.d_in)[self.r0:self.r1]
            self.blocks.append(O.Block(signs=O.pack_signs(sm), u=np.asarray(u[i][self.r0:self.r1], np.float64),
                                       v=np.asarray(v[i], np.float64)))
        self.n = len(self.blocks)

    def set_num_blocks(self, n):
        self.n = n

    def matmul(self, x):
        y = O.matmul_dense(self.blocks, self.s, self.n, x.numpy().astype(np.float64))
        return torch.from_numpy(y)


def _worker(rank, world, port, d_out, d_in, n, batch, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    w = rng.standard_normal((d_out, d_in))
    s, blocks = O.compress(w, rng.standard_normal((64, d_in)), n, 4, dtype="f32")
    signs = np.stack([b.signs for b in blocks])
    u = np.stack([b.u for b in blocks])
    v = np.stack([b.v for b in blocks])
    layer = TPLayer(d_out, d_in, k=4, n_capacity=n, factor_dtype="f32", local_factory=OracleShard, device=0)
    layer.load_blocks(0, signs, u, v, s)
    x = torch.from_numpy(rng.standard_normal((batch, d_in)))
    out = {}
    for level in range(n + 1):
        layer.set_num_blocks(level)
        y = layer.matmul(x)
        ref = O.matmul_dense(blocks, s, level, x.numpy())
        out[level] = float(np.max(np.abs(y.numpy() - ref)))
    results[rank] = out
    dist.destroy_process_group()


@pytest.mark.parametrize("d_out", [12, 13])   # even and uneven shards
def test_tp_world2_matches_unsharded(d_out):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, d_out, 9, 3, 2, results), nprocs=world, join=True)
    for rank in range(world):
        for level, err in results[rank].items():
            assert err <= 1e-12, (rank, level, err)


def test_shard_rows_cover_exactly():
    for d_out in (1, 7, 4096, 8191):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(d_out, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == d_out
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(8, 2, 2)


def _gather_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d_out, batch = 10, 3
    r0, r1 = shard_rows(d_out, world, rank)
    full = torch.arange(batch * d_out, dtype=torch.float32).reshape(batch, d_out)
    y = gather_rows(full[:, r0:r1].contiguous(), d_out)
    results[rank] = bool(torch.equal(y, full))
    dist.destroy_process_group()


def test_gather_rows_world3_uneven():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_gather_worker, args=(3, _free_port(), results), nprocs=3, join=True)
    assert all(results[r] for r in range(3))
