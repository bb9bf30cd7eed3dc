"""Row-sharded tensor parallelism for one BitStack layer.

Rank g of G owns output rows [g*d_out//G, (g+1)*d_out//G) of every block's S_i and U_i
(the library copies its shard inside bitstack_load_blocks); V_i and s are replicated.
Each rank runs bitstack_matmul on its rows with no communication inside the kernel; one
all-gather (NCCL over NVLink on B200, gloo in the CPU tests) assembles y [B, d_out].
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_rows(d_out: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced row range of `rank` (sizes differ by at most one row)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside [0, {world})")
    return d_out * rank // world, d_out * (rank + 1) // world


def gather_rows(y_local: torch.Tensor, d_out: int, group=None) -> torch.Tensor:
    """All-gather row slices y_local [B, r_g] of every rank into y [B, d_out].

    Shards may differ by one row: each rank pads to the largest shard, the padded
    [G, B, r_max] gather is reordered into [B, d_out] by copying each rank's rows."""
    world = dist.get_world_size(group)
    if y_local.is_cuda and dist.get_backend(group) == "gloo":
        # gloo has no device all-gather: stage through host memory (used by the CPU-plumbed
        # multi-process tests of the real library; NCCL moves device buffers directly)
        return gather_rows(y_local.cpu(), d_out, group).to(y_local.device)
    batch = y_local.shape[0]
    r_max = -(-d_out // world)
    if y_local.shape[1] < r_max:
        padded = torch.zeros((batch, r_max), dtype=y_local.dtype, device=y_local.device)
        padded[:, : y_local.shape[1]] = y_local
    else:
        padded = y_local.contiguous()
    flat = torch.empty((world * batch, r_max), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(flat, padded, group=group)   # concatenated along dim 0
    gathered = flat.view(world, batch, r_max)
    if d_out % world == 0:
        return gathered.permute(1, 0, 2).reshape(batch, d_out)
    y = torch.empty((batch, d_out), dtype=y_local.dtype, device=y_local.device)
    for g in range(world):
        r0, r1 = shard_rows(d_out, world, g)
        y[:, r0:r1] = gathered[g, :, : r1 - r0]
    return y


class TPLayer:
    """One BitStack layer row-sharded over the ranks of `group` (one process per GPU)."""

    def __init__(self, d_out: int, d_in: int, k: int = 16, n_capacity: int = 16, factor_dtype="bf16",
                 group=None, device: Optional[int] = None,
                 local_factory: Optional[Callable[..., object]] = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.d_out, self.d_in = d_out, d_in
        self.r0, self.r1 = shard_rows(d_out, self.world, self.rank)
        if local_factory is None:
            from .bitstack import Layer
            local_factory = Layer
        dev = torch.cuda.current_device() if device is None else device
        self.local = local_factory(d_out, d_in, k=k, n_capacity=n_capacity, factor_dtype=factor_dtype,
                                   row_begin=self.r0, row_end=self.r1, device=dev)

    def load_blocks(self, first_block: int, signs, u, v, s=None, stream=None) -> None:
        """Full-matrix buffers on every rank; the library keeps this rank's rows."""
        self.local.load_blocks(first_block, signs, u, v, s, stream=stream)

    def set_num_blocks(self, n: int) -> None:
        self.local.set_num_blocks(n)

    def matmul(self, x: torch.Tensor) -> torch.Tensor:
        y_local = self.local.matmul(x)
        if self.world == 1:
            return y_local
        return gather_rows(y_local, self.d_out, self.group)
