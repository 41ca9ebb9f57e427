"""Pins for the oracle's attention (Eq. 1, Eq. 27): brute-force numpy fp64 with the additive
mask materialised (an independent implementation of the definition), closed-form cases,
skipping exactness, convex hull, causality.  CPU only."""
import math

import numpy as np
import pytest


def _numpy_masked(q, k, v, scale, labels, T):
    """Materialised-M oracle: scores + additive mask (-inf on dropped tiles and on
    non-causal tokens), row softmax, times V — plain numpy fp64."""
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    m, n_c = Hq // Hkv, Nkv - Nq
    out = np.empty((Hq, Nq, C))
    t = np.arange(Nq)[:, None]
    s = np.arange(Nkv)[None, :]
    causal = s <= n_c + t
    for p in range(Hq):
        h = p // m
        sc = (q[p].astype(np.float64) @ k[h].astype(np.float64).T) * scale
        keep = causal.copy()
        if labels is not None:
            keep &= labels[h][t // T, s // T] > 0
        sc = np.where(keep, sc, -np.inf)
        w = np.exp(sc - sc.max(1, keepdims=True))
        out[p] = (w / w.sum(1, keepdims=True)) @ v[h].astype(np.float64)
    return out


def _rand(rng, Hq, Hkv, Nq, Nkv, C):
    f = lambda *s: rng.standard_normal(s).astype(np.float32)
    return f(Hq, Nq, C), f(Hkv, Nkv, C), f(Hkv, Nkv, C)


def _rand_labels(rng, orc, Hkv, Nq, Nkv, T, p=0.4):
    Tq, Tkv = -(-Nq // T), -(-Nkv // T)
    lab = (rng.random((Hkv, Tq, Tkv)) < p).astype(np.uint8)
    lab[:, :, 0] = 1  # sink column keeps every row non-empty
    for i in range(Tq):
        for j in range(Tkv):
            if not orc.causal(i, j, T, Nq, Nkv):
                lab[:, i, j] = 0
    return lab


@pytest.mark.parametrize("m,Nq,Nkv,C", [(1, 64, 64, 8), (2, 100, 100, 16), (4, 70, 200, 8), (2, 1, 1, 4)])
def test_dense_matches_bruteforce(orc, m, Nq, Nkv, C):
    rng = np.random.default_rng(m * 100 + Nq)
    q, k, v = _rand(rng, 2 * m, 2, Nq, Nkv, C)
    O, lse = orc.masked_attention(q, k, v, 1 / math.sqrt(C))
    ref = _numpy_masked(q, k, v, 1 / math.sqrt(C), None, 64)
    assert np.abs(O - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("seed", range(6))
def test_masked_matches_materialised(orc, seed):
    # streaming kernel == materialised-M oracle on random (workload, mask) pairs
    rng = np.random.default_rng(seed)
    m = [1, 2, 4][seed % 3]
    Nq = int(rng.integers(1, 300))
    Nkv = Nq + int(rng.integers(0, 200)) * (seed % 2)
    T = [16, 32, 64][seed % 3]
    q, k, v = _rand(rng, 2 * m, 2, Nq, Nkv, 8)
    lab = _rand_labels(rng, orc, 2, Nq, Nkv, T)
    O, _ = orc.masked_attention(q, k, v, 0.3, lab, T)
    ref = _numpy_masked(q, k, v, 0.3, lab, T)
    assert np.abs(O - ref).max() <= 1e-12


def test_keep_all_labels_equal_dense(orc):
    rng = np.random.default_rng(9)
    q, k, v = _rand(rng, 4, 2, 130, 130, 8)
    lab = _rand_labels(rng, orc, 2, 130, 130, 32, p=1.0)
    O1, l1 = orc.masked_attention(q, k, v, 0.25, lab, 32)
    O2, l2 = orc.masked_attention(q, k, v, 0.25)
    assert np.array_equal(O1, O2) and np.array_equal(l1, l2)


def test_single_token_and_constant_scores(orc):
    rng = np.random.default_rng(10)
    q, k, v = _rand(rng, 1, 1, 1, 1, 8)
    O, _ = orc.masked_attention(q, k, v, 0.5)
    assert np.array_equal(O[0, 0], v[0, 0].astype(np.float64))
    # q = 0 -> uniform softmax over the causal prefix -> running mean of V
    q = np.zeros((1, 40, 8), np.float32)
    k = rng.standard_normal((1, 60, 8)).astype(np.float32)
    v = rng.standard_normal((1, 60, 8)).astype(np.float32)
    O, lse = orc.masked_attention(q, k, v, 0.5)
    for t in range(40):
        assert np.allclose(O[0, t], v[0, : 20 + t + 1].astype(np.float64).mean(0), atol=1e-12)
        assert lse[0, t] == pytest.approx(math.log(20 + t + 1), abs=1e-12)


def test_skipping_exactness_and_hull(orc):
    # dropped tiles' K/V never matter; outputs are convex combinations of V rows
    rng = np.random.default_rng(11)
    Nq = Nkv = 256
    T = 32
    q, k, v = _rand(rng, 2, 1, Nq, Nkv, 8)
    lab = _rand_labels(rng, orc, 1, Nq, Nkv, T, p=0.3)
    O, _ = orc.masked_attention(q, k, v, 0.4, lab, T)
    k2, v2 = k.copy(), v.copy()
    dropped_cols = [j for j in range(Nkv // T) if not lab[0, :, j].any()]
    for j in dropped_cols:
        k2[:, j * T:(j + 1) * T] = 77.0
        v2[:, j * T:(j + 1) * T] = -55.0
    O2, _ = orc.masked_attention(q, k2, v2, 0.4, lab, T)
    assert np.array_equal(O, O2)
    lo, hi = v.min(1)[0], v.max(1)[0]
    assert (O >= lo - 1e-12).all() and (O <= hi + 1e-12).all()


def test_causality_perturbation(orc):
    # perturbing K/V beyond absolute position N_c + t never changes rows <= t
    rng = np.random.default_rng(12)
    Nq, Nkv = 96, 160
    q, k, v = _rand(rng, 2, 1, Nq, Nkv, 8)
    lab = _rand_labels(rng, orc, 1, Nq, Nkv, 32, p=0.6)
    O, _ = orc.masked_attention(q, k, v, 0.4, lab, 32)
    for t in [0, 17, 50, 95]:
        k2, v2 = k.copy(), v.copy()
        k2[:, Nkv - Nq + t + 1:] = rng.standard_normal(k2[:, Nkv - Nq + t + 1:].shape)
        v2[:, Nkv - Nq + t + 1:] = 9.0
        O2, _ = orc.masked_attention(q, k2, v2, 0.4, lab, 32)
        assert np.array_equal(O[:, : t + 1], O2[:, : t + 1])


def test_row_subset_matches_full(orc):
    rng = np.random.default_rng(13)
    q, k, v = _rand(rng, 4, 2, 100, 100, 8)
    O, lse = orc.masked_attention(q, k, v, 0.3)
    rows = np.array([[0, 0], [3, 99], [1, 50]])
    Os, ls = orc.masked_attention(q, k, v, 0.3, rows=rows)
    for r, (p, t) in enumerate(rows):
        assert np.array_equal(Os[r], O[p, t]) and ls[r] == lse[p, t]
