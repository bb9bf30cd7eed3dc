"""Memory-budget level selection for a set of weight stacks (host logic, no kernels).

BitStack's point is that the model's size follows the memory it is given: residual blocks are
loaded while the budget allows and offloaded in reverse order when it shrinks (Fig.2,
P:140). Which stacks get the next block is the paper's "Average" ordering: no stack
loads its (i+1)-th block before every stack has loaded its i-th, and within a level the stacks
receive their next block in an importance order (the paper ranks them by calibration
perplexity, which needs a real model; here the order is an input, e.g. a seeded permutation as
in the C4 bench).  Block sizes follow Eq.9, computed by the library.

The general form is the paper's *universal stack* (P:140): one sequence of (stack, block)
entries, loaded as a prefix while memory allows and offloaded from the end.  `universal_stack`
builds it for the three sortings the paper compares: Average (above), Random (a seeded
uniform shuffle of the universal stack) and Greedy (per (stack, level) importance scores --
perplexities in the paper, inputs here -- merged best-first).  A stack's block i+1 always
follows its block i (Eq.8 is a prefix sum), so every prefix is a valid set of levels.
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


def universal_stack(n_blocks: Sequence[int], kind: str = "average", order=None, scores=None,
                    seed: int = 0) -> list:
    """The universal residual stack (Alg.1 lines 24-44) as a list of (stack m, block i).

    n_blocks[m]: blocks stack m holds.  kind:
      "average" -- level by level (no stack loads block i+1 before every stack has loaded
                   block i); within level i the order is `order` (one permutation for every
                   level, or a list of per-level permutations), else ascending scores[m][i]
                   (lower perplexity = more important = loaded first), else index order;
      "random"  -- a seeded uniform shuffle of the whole stack ("Random"), kept valid by
                   giving stack m its blocks in order at its successive positions;
      "greedy"  -- scores[m][i] = importance of stack m at level i+1 measured with every other
                   stack at n/2 ("Greedy"); entries are taken best-first (lowest score)
                   among the stacks' next blocks (reading R23: the precedence i before i+1 is
                   kept, so a stack's later block waits for its earlier one).
    """
    n_m = len(n_blocks)
    nb = [int(b) for b in n_blocks]
    if any(b < 0 for b in nb):
        raise ValueError("n_blocks must be >= 0")
    if kind == "average":
        out = []
        for i in range(max(nb, default=0)):
            if order is not None:
                per_level = len(order) > 0 and hasattr(order[0], "__len__")
                lvl = [int(m) for m in (order[i] if per_level else order)]
                if sorted(lvl) != list(range(n_m)):
                    raise ValueError("order must be a permutation of the stack indices")
            elif scores is not None:
                lvl = sorted(range(n_m), key=lambda m: (float(scores[m][i]) if i < nb[m] else 0.0, m))
            else:
                lvl = list(range(n_m))
            out.extend((m, i) for m in lvl if i < nb[m])
        return out
    if kind == "random":
        import numpy as np
        seq = np.random.default_rng(seed).permutation(np.repeat(np.arange(n_m), nb))
        nxt = [0] * n_m
        out = []
        for m in seq.tolist():
            out.append((m, nxt[m]))
            nxt[m] += 1
        return out
    if kind == "greedy":
        if scores is None:
            raise ValueError("greedy needs scores[m][i]")
        import heapq
        heap = [(float(scores[m][0]), m, 0) for m in range(n_m) if nb[m] > 0]
        heapq.heapify(heap)
        out = []
        while heap:
            _, m, i = heapq.heappop(heap)
            out.append((m, i))
            if i + 1 < nb[m]:
                heapq.heappush(heap, (float(scores[m][i + 1]), m, i + 1))
        return out
    raise ValueError(f"unknown sorting {kind!r} (average | random | greedy)")


def prefix_levels(stack: Sequence, sizes: Sequence[float], budget: float) -> list:
    """Per-stack levels of the longest prefix of the universal stack that fits `budget` bytes
    (blocks are pushed from the top until the next one does not fit)."""
    levels = [0] * len(sizes)
    used = 0.0
    for m, i in stack:
        if i != levels[m]:
            raise ValueError("universal stack out of order: block %d of stack %d before block %d" % (i, m, levels[m]))
        if used + sizes[m] > budget:
            break
        used += sizes[m]
        levels[m] += 1
    return levels


class StackSet:
    """A set of Layer handles whose levels follow one memory budget (bitstack_set_num_blocks on
    each; blocks above a stack's level stay resident and are simply not used).  `kind`, `order`,
    `scores`, `seed` choose the universal stack's sorting (`universal_stack`); the default is
    the paper's Average ordering over the blocks every handle holds."""

    def __init__(self, layers, order: Optional[Sequence[int]] = None, factor_bits: int = 16,
                 kind: str = "average", scores=None, seed: int = 0):
        self.layers = list(layers)
        self.order = order
        self.sizes = [block_bytes(l.d_out, l.d_in, l.k, factor_bits) for l in self.layers]
        self.kind, self.scores, self.seed = kind, scores, seed

    def levels_for(self, budget: float) -> list:
        resident = [l.info()["n_resident"] for l in self.layers]
        if self.kind == "average" and self.scores is None:
            return average_levels(self.sizes, budget, self.order, max_level=min(resident, default=0))
        stack = universal_stack(resident, self.kind, self.order, self.scores, self.seed)
        return prefix_levels(stack, self.sizes, budget)

    def apply_budget(self, budget: float) -> list:
        levels = self.levels_for(budget)
        for lay, n in zip(self.layers, levels):
            lay.set_num_blocks(n)
        return levels
