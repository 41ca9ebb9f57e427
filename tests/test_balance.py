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


# ---- split-KV piece planner (parallel.plan_pieces, §8 f2) ---------------------------------------
def _diffuse_counts(seed, B=1, H=8, tq=256, dense_heads=1):
    """Kept tiles per row: causal extent i + 1; dense_heads diffuse heads keep ~40 %, the others ~8 %
    plus a band of 8 (the structured-input shape)."""
    rng = np.random.default_rng(seed)
    c = np.zeros((B, H, tq), dtype=np.int32)
    for r in range(B):
        for h in range(H):
            kap = 0.4 if h < dense_heads else 0.08
            n = np.arange(1, tq + 1)
            c[r, h] = np.minimum(n, (kap * n + 8 + rng.integers(0, 4, tq)).astype(np.int64))
    return c


@pytest.mark.parametrize("parts", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("dense_heads,B", [(0, 1), (1, 1), (3, 1), (1, 2)])
def test_plan_pieces_covers_every_tile_once(parts, dense_heads, B):
    from paper_2605_12193_b200 import parallel

    counts = _diffuse_counts(parts + dense_heads, B=B, dense_heads=dense_heads)
    plan = parallel.plan_pieces(counts, parts)
    kept, ext = parallel._lpt_rows(counts)
    assert len(plan) == parts
    whole = np.zeros(len(kept), dtype=np.int64)
    runs = {}
    for r, pieces in enumerate(plan):
        for r0, r1, a, b, slot in pieces:
            assert 0 <= r0 < r1 <= len(kept)
            if (a, b) == (0, 0):
                assert slot == 0
                whole[r0:r1] += 1
            else:
                runs.setdefault((r0, r1), []).append((a, b, slot, r))
    covered = whole.copy()
    for (r0, r1), rng_ in runs.items():
        rng_.sort()
        # the KV ranges of a run partition [0, tkv_run) without gaps or overlap, reach every row's
        # causal extent, sit in distinct partial slots and on distinct ranks (they run concurrently)
        assert rng_[0][0] == 0 and all(x[1] == y[0] for x, y in zip(rng_, rng_[1:]))
        assert rng_[-1][1] >= ext[r0:r1].max()
        assert sorted(x[2] for x in rng_) == list(range(len(rng_)))
        assert len({x[3] for x in rng_}) == len(rng_)
        covered[r0:r1] += 1
    assert (covered == 1).all(), "every row exactly once: as a whole row or as one split run"
    assert parallel.plan_slots(plan) == 1 + max([len(v) - 1 for v in runs.values()], default=0)


def test_plan_pieces_splits_only_rows_above_the_per_sm_share():
    from paper_2605_12193_b200 import parallel

    counts = _diffuse_counts(3, dense_heads=1, tq=512)
    kept, ext = parallel._lpt_rows(counts)
    cost = kept + 3
    # few ranks: every row fits one rank's per-SM share -> plain row slices (bfla_balance_rows' job)
    for parts in (1, 2, 4):
        assert all((p[2], p[3]) == (0, 0) for pl in parallel.plan_pieces(counts, parts) for p in pl)
    plan = parallel.plan_pieces(counts, 8)
    share = -(-int(cost.sum()) // (8 * 148))
    split_rows = {x for pl in plan for p in pl if p[3] for x in range(p[0], p[1])}
    assert set(np.nonzero(cost > share)[0].tolist()) <= split_rows
    tq = counts.shape[-1]
    for x in split_rows:  # a run starts at its head's first (longest) row and is contiguous
        assert all(y in split_rows for y in range(x - x % tq, x))
    # the longest piece estimate is near the per-SM share (a split row's ranges share its tiles)
    for pl in plan:
        for r0, r1, a, b, _ in pl:
            if b:
                est = max(kept[x] * max(0, min(b, ext[x]) - a) / ext[x] for x in range(r0, r1)) + 3
                assert est <= 2 * share
    # rank loads stay within one share of the ideal
    loads = []
    for pl in plan:
        L = 0.0
        for r0, r1, a, b, _ in pl:
            L += cost[r0:r1].sum() if not b else sum(kept[x] * max(0, min(b, ext[x]) - a) / ext[x] + 3
                                                     for x in range(r0, r1))
        loads.append(L)
    assert max(loads) <= cost.sum() / 8 + 2 * share
