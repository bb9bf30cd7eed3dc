"""Memory-budget level selection for a set of weight stacks (host logic, no kernels).

BitStack's point is that the model's size follows the memory it is given: residual blocks are
loaded while the budget allows and offloaded in reverse order when it shrinks (Fig.2,
P:140). Which stacks get the next block is the paper's "Average" ordering: no stack
loads its (i+1)-th block before every stack has loaded its i-th, and within a level the stacks
receive their next block in an importance order (the paper ranks them by calibration
perplexity, which needs a real model; here the order is an input, e.g. a seeded permutation as
in the C4 bench).  Block sizes follow Eq.9, computed by the library.
"""
from __future__ import annotations

from typing import Optional, Sequence


def block_bytes(d_out: int, d_in: int, k: int = 16, factor_bits: int = 16) -> float:
    """Stored size of one residual block in bytes (Eq.9 / 8), via bitstack_block_size_bits."""
    from .bitstack import block_size_bits
    return block_size_bits(d_out, d_in, k, factor_bits) / 8.0


def average_levels(sizes: Sequence[float], budget: float, order: Optional[Sequence[int]] = None,
                   max_level: Optional[int] = None) -> list:
    """Per-stack block counts under `budget` (bytes) with the Average ordering.

    sizes[m]: bytes of one block of stack m.  Whole levels are added while every stack's next
    block fits; the last, partial level goes to the stacks in `order` (default: index order)
    until the next one in that order no longer fits.  `max_level` caps the level (e.g. the
    blocks a stack holds).  The returned levels differ by at most 1 between stacks.
    """
    n_m = len(sizes)
    order = list(range(n_m)) if order is None else [int(m) for m in order]
    if sorted(order) != list(range(n_m)):
        raise ValueError("order must be a permutation of the stack indices")
    levels = [0] * n_m
    used = 0.0
    per_level = float(sum(sizes))
    level = 0
    while (max_level is None or level < max_level) and n_m:
        if used + per_level <= budget:
            levels = [lv + 1 for lv in levels]
            used += per_level
            level += 1
            continue
        for m in order:                 # the partial level, in importance order
            if used + sizes[m] > budget:
                break
            levels[m] += 1
            used += sizes[m]
        break
    return levels


class StackSet:
    """A set of Layer handles whose levels follow one memory budget (bitstack_set_num_blocks on
    each; blocks above a stack's level stay resident and are simply not used)."""

    def __init__(self, layers, order: Optional[Sequence[int]] = None, factor_bits: int = 16):
        self.layers = list(layers)
        self.order = order
        self.sizes = [block_bytes(l.d_out, l.d_in, l.k, factor_bits) for l in self.layers]

    def levels_for(self, budget: float) -> list:
        cap = min((l.info()["n_resident"] for l in self.layers), default=0)
        return average_levels(self.sizes, budget, self.order, max_level=cap)

    def apply_budget(self, budget: float) -> list:
        levels = self.levels_for(budget)
        for lay, n in zip(self.layers, levels):
            lay.set_num_blocks(n)
        return levels
