"""§8 f2 host logic: the cost-balanced row partition (bfla_balance_rows, a host-only entry point of
libbfla.so) against brute force over every contiguous partition of small inputs."""
import itertools

import numpy as np
import pytest

import paper_2605_12193_b200 as bf


def _lpt_costs(counts, overhead):
    """Row costs in the LPT order rho = (r*H + h)*Tq + (Tq-1-i) (include/bfla.h)."""
    B, H, Tq = counts.shape
    return [int(counts[r, h, Tq - 1 - i]) + overhead for r in range(B) for h in range(H) for i in range(Tq)]


def _best_bottleneck(costs, parts):
    n = len(costs)
    best = sum(costs)
    for cuts in itertools.combinations_with_replacement(range(n + 1), parts - 1):
        b = (0,) + cuts + (n,)
        best = min(best, max(sum(costs[b[k]:b[k + 1]]) for k in range(parts)))
    return best


@pytest.mark.parametrize("seed", range(12))
def test_balance_rows_is_optimal_and_valid(seed):
    rng = np.random.default_rng(seed)
    B, H, Tq = int(rng.integers(1, 3)), int(rng.integers(1, 3)), int(rng.integers(1, 5))
    counts = rng.integers(0, 40, size=(B, H, Tq)).astype(np.int32)
    overhead = int(rng.integers(0, 4))
    n = B * H * Tq
    costs = _lpt_costs(counts, overhead)
    for parts in (1, 2, 3, 5):
        bounds = bf.bfla_balance_rows(counts, parts, overhead)
        assert len(bounds) == parts + 1 and bounds[0] == 0 and bounds[-1] == n
        assert all(a <= b for a, b in zip(bounds, bounds[1:]))
        if n >= parts:
            assert all(a < b for a, b in zip(bounds, bounds[1:])), "empty slice although rows remain"
        got = max(sum(costs[a:b]) for a, b in zip(bounds, bounds[1:]))
        assert got == _best_bottleneck(costs, parts), (bounds, costs)


def test_balance_rows_uses_lpt_order():
    # one request, one head, Tq = 4: LPT order visits i = 3, 2, 1, 0; a heavy last row must sit alone
    counts = np.array([[[1, 1, 1, 30]]], dtype=np.int32)
    assert bf.bfla_balance_rows(counts, 2, 0) == [0, 1, 4]


def test_balance_rows_head_skew():
    """Per-head kappa skew: equal head counts per part are not equal work; the balanced cut splits
    the heavy head across parts (the §8 f2 motivation)."""
    rng = np.random.default_rng(3)
    Tq = 64
    causal = np.arange(1, Tq + 1)
    dens = np.array([0.9, 0.1, 0.1, 0.1])  # one dense head
    counts = np.maximum(1, (causal[None, :] * dens[:, None]).astype(np.int32))[None]
    costs = _lpt_costs(counts, 3)
    per_head = [sum(costs[h * Tq:(h + 1) * Tq]) for h in range(4)]
    bounds = bf.bfla_balance_rows(counts, 4, 3)
    parts = [sum(costs[a:b]) for a, b in zip(bounds, bounds[1:])]
    assert max(parts) < 0.6 * max(per_head)
    assert max(parts) <= sum(costs) / 4 + max(costs)  # within one row of perfect balance


def test_balance_rows_rejects_bad_arguments():
    with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
        bf.bfla_balance_rows(np.zeros((1, 1, 4), np.int32), 0)
    with pytest.raises(ValueError):
        bf.bfla_balance_rows(np.zeros((4,), np.int32), 2)
