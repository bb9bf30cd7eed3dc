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
