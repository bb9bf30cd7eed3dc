"""Memory-budget level selection (paper_2410_23918_b200/budget.py): the Average ordering's
invariants, and the paper's own 8B memory points (P:177-217 budgets; one level of
all 224 Llama-3.1-8B matrices is 912 MiB on top of 2004.5 MiB of embeddings / head / norms)."""
import numpy as np
import pytest

from synthetic import C4_LEVELS, LLAMA31_8B_SHAPES


@pytest.fixture(scope="module")
def budget_mod():
    from paper_2410_23918_b200 import build as B
    B.build()
    from paper_2410_23918_b200 import budget
    return budget


def test_average_levels_invariants(budget_mod):
    rng = np.random.default_rng(0)
    sizes = rng.uniform(1.0, 10.0, 37).tolist()
    order = rng.permutation(37).tolist()
    prev = None
    for budget in np.linspace(0, 5 * sum(sizes), 41):
        lv = budget_mod.average_levels(sizes, float(budget), order)
        assert max(lv) - min(lv) <= 1                                   # Average: spread <= 1
        assert sum(l * s for l, s in zip(lv, sizes)) <= budget + 1e-9    # fits
        if prev is not None:
            assert all(a >= b for a, b in zip(lv, prev))                # monotone in the budget
        hi = [m for m in order if lv[m] == max(lv)] if max(lv) != min(lv) else []
        assert hi == order[:len(hi)]                                    # partial level = prefix of the order
        prev = lv
    assert budget_mod.average_levels(sizes, 1e9, order, max_level=3) == [3] * 37
    with pytest.raises(ValueError):
        budget_mod.average_levels([1.0, 2.0], 5.0, [0, 0])


def test_llama31_8b_memory_points(budget_mod):
    """The paper's 8B budgets map to the average levels SURVEY §8(d) derives for config C4."""
    sizes = [budget_mod.block_bytes(*LLAMA31_8B_SHAPES[name]) for _ in range(32) for name in LLAMA31_8B_SHAPES]
    assert abs(sum(sizes) / 2 ** 20 - 912.0) < 0.5                      # one level of the whole model
    order = np.random.default_rng(4).permutation(len(sizes)).tolist()
    for budget_mib, level in C4_LEVELS.items():
        lv = budget_mod.average_levels(sizes, (budget_mib - 2004.5) * 2 ** 20, order)
        loaded = sum(l * s for l, s in zip(lv, sizes)) / sum(sizes)      # levels in model-size units
        assert abs(loaded - level) < 0.01, (budget_mib, loaded, level)
        assert max(lv) - min(lv) == 1 and min(lv) == int(level)


# ------------------------------------------------------------------ the universal stack
def _valid(stack, n_blocks):
    """every (m, i) exactly once, and stack m's blocks in order 0, 1, 2, ..."""
    nxt = [0] * len(n_blocks)
    for m, i in stack:
        assert i == nxt[m]
        nxt[m] += 1
    assert nxt == list(n_blocks)


def test_universal_stack_average_is_average_levels(budget_mod):
    """The Average universal stack's prefixes are exactly average_levels."""
    rng = np.random.default_rng(1)
    sizes = rng.uniform(1.0, 10.0, 23).tolist()
    order = rng.permutation(23).tolist()
    stack = budget_mod.universal_stack([6] * 23, "average", order)
    _valid(stack, [6] * 23)
    for budget in np.linspace(0, 7 * sum(sizes), 57) + 0.37:   # off the exact level boundaries
        assert budget_mod.prefix_levels(stack, sizes, float(budget)) == \
            budget_mod.average_levels(sizes, float(budget), order, max_level=6)


def test_universal_stack_average_per_level_scores(budget_mod):
    """Within level i the blocks are sorted by their measured score (lower perplexity first,
    P:146: 'blocks with lower measured perplexity scores are on top')."""
    scores = [[3.0, 1.0], [1.0, 2.0], [2.0, 3.0]]
    assert budget_mod.universal_stack([2, 2, 2], "average", scores=scores) == \
        [(1, 0), (2, 0), (0, 0), (0, 1), (1, 1), (2, 1)]
    per_level = [[2, 0, 1], [1, 2, 0]]
    assert budget_mod.universal_stack([2, 2, 2], "average", per_level) == \
        [(2, 0), (0, 0), (1, 0), (1, 1), (2, 1), (0, 1)]
    assert budget_mod.universal_stack([1, 3], "average") == [(0, 0), (1, 0), (1, 1), (1, 2)]   # ragged


def test_universal_stack_random(budget_mod):
    """Random: a seeded shuffle, valid, reproducible; its levels are NOT balanced."""
    nb = [16] * 224
    a = budget_mod.universal_stack(nb, "random", seed=3)
    _valid(a, nb)
    assert a == budget_mod.universal_stack(nb, "random", seed=3)
    assert a != budget_mod.universal_stack(nb, "random", seed=4)
    lv = budget_mod.prefix_levels(a, [1.0] * 224, 224 * 4)
    assert sum(lv) == 224 * 4 and max(lv) - min(lv) > 1
    # uniform interleaving: the first entry is each stack with equal probability
    firsts = np.bincount([budget_mod.universal_stack([2] * 4, "random", seed=s)[0][0] for s in range(4000)],
                         minlength=4)
    assert firsts.min() > 850 and firsts.max() < 1150


def test_universal_stack_greedy(budget_mod):
    """Greedy: best score first among the stacks' next blocks, checked step by step on a
    hand-worked case."""
    scores = [[5.0, 1.0, 9.0], [2.0, 8.0, 3.0], [4.0, 0.5, 7.0]]
    got = budget_mod.universal_stack([3, 3, 3], "greedy", scores=scores)
    _valid(got, [3, 3, 3])
    # at every step the lowest score among the stacks' next blocks
    want = []
    nxt = [0, 0, 0]
    for _ in range(9):
        cand = [(scores[m][nxt[m]], m) for m in range(3) if nxt[m] < 3]
        _, m = min(cand)
        want.append((m, nxt[m]))
        nxt[m] += 1
    assert got == want == [(1, 0), (2, 0), (2, 1), (0, 0), (0, 1), (2, 2), (1, 1), (1, 2), (0, 2)]
    with pytest.raises(ValueError):
        budget_mod.universal_stack([3, 3, 3], "greedy")
    with pytest.raises(ValueError):
        budget_mod.universal_stack([3], "bogus")


def test_prefix_levels_nested_and_fits(budget_mod):
    """Loading more memory only adds blocks (the nested property that makes BitStack's size
    continuous), for every sorting; the loaded bytes never exceed the budget."""
    rng = np.random.default_rng(7)
    nb = rng.integers(0, 9, 31).tolist()
    sizes = rng.uniform(1.0, 5.0, 31).tolist()
    scores = rng.uniform(0, 1, (31, 9)).tolist()
    for kind in ("average", "random", "greedy"):
        stack = budget_mod.universal_stack(nb, kind, scores=scores if kind != "random" else None, seed=5)
        _valid(stack, nb)
        prev = [0] * 31
        for budget in np.linspace(0, sum(b * s for b, s in zip(nb, sizes)) + 1, 40):
            lv = budget_mod.prefix_levels(stack, sizes, float(budget))
            assert all(a >= b for a, b in zip(lv, prev)) and all(l <= b for l, b in zip(lv, nb))
            assert sum(l * s for l, s in zip(lv, sizes)) <= budget + 1e-9
            prev = lv
        assert prev == nb
    with pytest.raises(ValueError):
        budget_mod.prefix_levels([(0, 1)], [1.0], 5.0)
