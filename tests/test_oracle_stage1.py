"""Pins for the oracle's Stage 1 (Eq. 4-18): closed forms, worked examples, brute force on
integer-valued inputs (where fp32 arithmetic is exact, so a numpy int64 computation is an
independent exact reference), textbook reductions and invariants.  CPU only."""
import math

import numpy as np
import pytest


def _int_inputs(rng, H, N, C, lo=-3, hi=4):
    return rng.integers(lo, hi, size=(H, N, C)).astype(np.float32)


# ---------------------------------------------------------------- Eq. 11-13
def test_causal_block_mask_square(orc):
    # N_q = N_kv = 4b, N_c = 0 -> lower-triangular incl. diagonal
    b = 8
    M = np.array([[orc.causal(i, j, b, 4 * b, 4 * b) for j in range(4)] for i in range(4)])
    assert (M == np.tril(np.ones((4, 4), bool))).all()


def test_causal_block_mask_chunked(orc):
    # N_q = b, N_kv = 3b (N_c = 2b): e_0 = 3b-1 >= p_2 = 2b -> all 3 KV blocks causal
    b = 16
    assert [orc.causal(0, j, b, b, 3 * b) for j in range(3)] == [True, True, True]
    # N_q = N_kv = 1, b = 256 -> 1x1 mask = 1
    assert orc.causal(0, 0, 256, 1, 1)


def test_causal_tiles_count(orc):
    assert orc.causal_tiles(2048, 2048, 64) == 32 * 33 // 2
    # ragged: N = 100, T = 64 -> tiles 2x2, causal: (0,0),(1,0),(1,1)
    assert orc.causal_tiles(100, 100, 64) == 3
    # chunked: Nq = 64, Nkv = 192 -> one row, all 3 tiles causal
    assert orc.causal_tiles(64, 192, 64) == 3


# ---------------------------------------------------------------- Eq. 4-7
def test_flatten_spec_example(orc):
    # N=5, b=4, g=2, C=1, X=[1..5] -> block 0 ([1,2],[3,4]); block 1 ([5,0],[0,0]); valid [2,1]
    x = np.arange(1, 6, dtype=np.float32).reshape(1, 5, 1)
    phi, valid = orc.flatten(x, 4, 2)
    assert phi.shape == (1, 2, 2, 2)
    assert phi[0, 0].tolist() == [[1, 2], [3, 4]]
    assert phi[0, 1].tolist() == [[5, 0], [0, 0]]
    assert valid.sum(1).tolist() == [2, 1]


def test_flatten_roundtrip(orc):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 77, 5)).astype(np.float32)
    phi, _ = orc.flatten(x, 16, 4)
    back = phi.reshape(3, -1, 4, 5).reshape(3, -1, 5)[:, :77]  # (l, u, t) -> token order
    assert np.array_equal(back, x)


# ---------------------------------------------------------------- Eq. 9-10
def _brute_block_scores_exact(q, k, b, g, m):
    """Eq. 9-10 by brute force in int64 (inputs integer-valued): group-pair dot products are
    sums of token dot products; block score = max over valid group pairs (causal only)."""
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    Lq, Lkv, G = -(-Nq // b), -(-Nkv // b), b // g
    n_c = Nkv - Nq
    qi, ki = q.astype(np.int64), k.astype(np.int64)
    S = np.full((Hq, Lq, Lkv), -np.inf)
    for p in range(Hq):
        QK = qi[p] @ ki[p // m].T  # token-level dot products [Nq, Nkv]
        for i in range(Lq):
            for j in range(Lkv):
                if j * b > min(n_c + (i + 1) * b - 1, Nkv - 1):
                    continue
                best = None
                for u in range(G):
                    t0 = i * b + u * g
                    if t0 >= Nq:
                        continue
                    for v in range(G):
                        s0 = j * b + v * g
                        if s0 >= Nkv:
                            continue
                        # flattened group dot = sum over aligned token offsets (t, s0 + t - t0)
                        tot = 0
                        for o in range(g):
                            if t0 + o < Nq and s0 + o < Nkv:
                                tot += QK[t0 + o, s0 + o]
                        best = tot if best is None else max(best, tot)
                S[p, i, j] = best
    return S


@pytest.mark.parametrize("Nq,Nkv,b,g,m", [(64, 64, 16, 4, 2), (50, 50, 16, 8, 1), (40, 72, 16, 4, 4),
                                         (64, 64, 16, 16, 2), (64, 64, 16, 1, 1)])
def test_block_scores_exact_on_integers(orc, Nq, Nkv, b, g, m):
    rng = np.random.default_rng(Nq * 7 + g)
    q = _int_inputs(rng, 2 * m, Nq, 8)
    k = _int_inputs(rng, 2, Nkv, 8)
    S = orc.block_scores(q, k, b, g)
    ref = _brute_block_scores_exact(q, k, b, g, m)
    assert np.array_equal(S, ref.astype(np.float32))


def test_block_scores_g1_is_block_max_of_qkT(orc):
    # g = 1: every group is one token -> S = max over the b x b block of Q K^T (textbook)
    rng = np.random.default_rng(1)
    q = _int_inputs(rng, 2, 64, 16)
    k = _int_inputs(rng, 1, 64, 16)
    S = orc.block_scores(q, k, 16, 1)
    QK = q.astype(np.int64) @ k[0].astype(np.int64).T  # [2, 64, 64]
    blk = QK.reshape(2, 4, 16, 4, 16).max(axis=(2, 4)).astype(np.float32)
    tri = np.tril(np.ones((4, 4), bool))
    assert np.array_equal(S[:, tri], blk[:, tri])
    assert np.isneginf(S[:, ~tri]).all()


def test_block_scores_gb_is_diagonal_trace(orc):
    # g = b: G = 1, the single group pair = trace of the b x b block of Q K^T
    rng = np.random.default_rng(2)
    q = _int_inputs(rng, 1, 64, 8)
    k = _int_inputs(rng, 1, 64, 8)
    S = orc.block_scores(q, k, 16, 16)
    QK = q[0].astype(np.int64) @ k[0].astype(np.int64).T
    for i in range(4):
        for j in range(i + 1):
            assert S[0, i, j] == np.trace(QK[16 * i:16 * i + 16, 16 * j:16 * j + 16])


def test_block_scores_float_close_to_exact(orc):
    # general floats: the canonical fp32 chain is within the textbook bound gamma_n * sum|xy|
    rng = np.random.default_rng(3)
    q = rng.standard_normal((2, 128, 32)).astype(np.float32)
    k = rng.standard_normal((1, 128, 32)).astype(np.float32)
    S = orc.block_scores(q, k, 32, 8)
    G, gc = 4, 8 * 32
    pq = q.reshape(2, 4, G, gc).astype(np.float64)
    pk = k.reshape(1, 4, G, gc).astype(np.float64)
    for p in range(2):
        for i in range(4):
            for j in range(i + 1):
                prods = pq[p, i][:, None, :] * pk[0, j][None, :, :]
                exact = prods.sum(-1)
                bound = gc * 2.0 ** -24 / (1 - gc * 2.0 ** -24) * np.abs(prods).sum(-1)
                u, v = np.unravel_index(np.argmax(exact), exact.shape)
                assert abs(S[p, i, j] - exact.max()) <= bound.max() + 1e-6


def test_block_scores_two_level_order_bound(orc):
    # DESIGN.md §4 item 2: a group dot is g token dots (C-long FMA chains) added in token order, so
    # every product passes through at most C + g roundings: |S - exact| <= gamma_{C+g} sum|xy| — a
    # bound the single gC-long chain does not meet in general (tight inputs: large cancelling terms).
    rng = np.random.default_rng(13)
    C, g, b = 32, 16, 64
    q = (rng.standard_normal((1, 256, C)) * np.exp(rng.standard_normal((1, 256, C)) * 2)).astype(np.float32)
    k = (rng.standard_normal((1, 256, C)) * np.exp(rng.standard_normal((1, 256, C)) * 2)).astype(np.float32)
    S = orc.block_scores(q, k, b, g)
    G, gc = b // g, g * C
    pq = q.reshape(1, 4, G, gc).astype(np.float64)
    pk = k.reshape(1, 4, G, gc).astype(np.float64)
    n = C + g
    for i in range(4):
        for j in range(i + 1):
            prods = pq[0, i][:, None, :] * pk[0, j][None, :, :]
            exact = prods.sum(-1)
            bound = n * 2.0 ** -24 / (1 - n * 2.0 ** -24) * np.abs(prods).sum(-1)
            # the max over pairs moves by at most the largest per-pair bound
            assert abs(S[0, i, j] - exact.max()) <= bound.max()


def test_block_scores_linearity(orc):
    # scaling K block j by 2 doubles S[., ., j] (exact: power-of-two scale)
    rng = np.random.default_rng(4)
    q = rng.standard_normal((1, 64, 16)).astype(np.float32)
    k = rng.standard_normal((1, 64, 16)).astype(np.float32)
    S = orc.block_scores(q, k, 16, 4)
    k2 = k.copy()
    k2[:, 16:32] *= 2
    S2 = orc.block_scores(q, k2, 16, 4)
    assert np.array_equal(S2[:, 1:, 1], 2 * S[:, 1:, 1])
    # max of doubled scores = 2 * max when the block max is positive; negative max stays the max of 2x
    assert np.array_equal(S2[:, :, 0], S[:, :, 0])


def test_block_scores_mean_pool_integer(orc):
    # MEAN (R1): block means of integer tokens with power-of-two counts are exact dyadics
    rng = np.random.default_rng(5)
    q = _int_inputs(rng, 2, 64, 8)
    k = _int_inputs(rng, 1, 64, 8)
    S = orc.block_scores(q, k, 16, 16, orc.POOL_MEAN)
    qm = q.reshape(2, 4, 16, 8).mean(2).astype(np.float64)
    km = k.reshape(1, 4, 16, 8).mean(2).astype(np.float64)
    ref = np.einsum("pic,jc->pij", qm, km[0])
    tri = np.tril(np.ones((4, 4), bool))
    assert np.array_equal(S[:, tri], ref[:, tri].astype(np.float32))
    assert np.isneginf(S[:, ~tri]).all()


def test_block_scores_mean_pool_ragged_blocks(orc):
    # MEAN (R1, R3) on ragged tails: the mean of a partial block divides by its REAL token count
    # (5 and 3 here, not b = 16).  Integer tokens are built so every channel sum of a partial block is
    # a multiple of its count, so the means are exact integers and the scores exact (|S| << 2^24).
    rng = np.random.default_rng(6)

    def ragged(h, n, b, c):
        x = rng.integers(-3, 4, size=(h, n, c)).astype(np.float32)
        n_last = n % b
        tail = x[:, n - n_last:]
        target = rng.integers(-2, 3, size=(h, c)).astype(np.float32)
        tail[:, -1] = n_last * target - tail[:, :-1].sum(1)  # channel sum = n_last * target
        return x

    for nq, nkv in ((37, 37), (35, 51)):  # square ragged; chunked (N_c = 16) with different tails
        q = ragged(2, nq, 16, 8)
        k = ragged(1, nkv, 16, 8)
        S = orc.block_scores(q, k, 16, 16, orc.POOL_MEAN)
        Lq, Lkv, nc = -(-nq // 16), -(-nkv // 16), nkv - nq
        qm = np.stack([q[:, 16 * i:min(nq, 16 * i + 16)].astype(np.float64).mean(1) for i in range(Lq)], 1)
        km = np.stack([k[0, 16 * j:min(nkv, 16 * j + 16)].astype(np.float64).mean(0) for j in range(Lkv)], 0)
        # partial-block means are integers by construction; full-block means are dyadic (/16): all exact
        assert np.array_equal(qm[:, -1], np.round(qm[:, -1])) and np.array_equal(km[-1], np.round(km[-1]))
        ref = np.einsum("pic,jc->pij", qm, km)
        for i in range(Lq):
            e_i = min(nc + 16 * (i + 1) - 1, nkv - 1)  # Eq. 11-13
            for j in range(Lkv):
                if 16 * j <= e_i:
                    assert S[0, i, j] == ref[0, i, j] and S[1, i, j] == ref[1, i, j], (nq, nkv, i, j)
                else:
                    assert np.isneginf(S[:, i, j]).all()
        # the divisor matters: with b = 16 in place of the real count the last blocks would differ
        assert not np.allclose(k[0, 16 * (Lkv - 1):].sum(0) / 16, km[-1])


# ---------------------------------------------------------------- Eq. 15
def test_exp2_canon_accuracy(orc):
    ts = np.concatenate([np.linspace(-126, 0, 20001), -np.logspace(-8, 0, 500)]).astype(np.float32)
    for t in ts:
        e = orc.exp2_canon(float(t))
        ref = 2.0 ** float(t)
        assert abs(e - ref) <= 2 * np.spacing(np.float32(ref)), (t, e, ref)
    assert orc.exp2_canon(0.0) == 1.0
    assert orc.exp2_canon(-127.0) == 0.0
    assert orc.exp2_canon(-3.0) == 0.125


def test_block_softmax_examples(orc):
    # S:198-200
    assert orc.block_softmax_row([0.0, 0.0], 128).tolist() == [0.5, 0.5]
    assert orc.block_softmax_row([3.5], 128).tolist() == [1.0]
    A = orc.block_softmax_row([1.0, 2.0], 4)  # alpha = 1/2 -> softmax of [0.5, 1.0]
    ref = np.exp([0.5, 1.0]) / np.exp([0.5, 1.0]).sum()
    assert np.allclose(A, ref, rtol=3e-7, atol=0)
    A = orc.block_softmax_row([1.0, -np.inf, 1.0], 4)
    assert A.tolist() == [0.5, 0.0, 0.5]


def test_block_softmax_matches_double(orc):
    rng = np.random.default_rng(6)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        s = (rng.standard_normal(n) * 200).astype(np.float32)
        A = orc.block_softmax_row(s, 128)
        x = s.astype(np.float64) / math.sqrt(128)
        ref = np.exp(x - x.max())
        ref /= ref.sum()
        assert np.abs(A - ref).max() <= 1e-6
        assert abs(A.astype(np.float64).sum() - 1) <= n * 2 ** -23


# ---------------------------------------------------------------- Eq. 16-18
def test_keep_select_spec_examples(orc):
    # [0.5, 0.3, 0.15, 0.05], gamma = 0.9 -> keep {0, 1, 2}
    keep, r, km, pp, tie = orc.keep_select([0.5, 0.3, 0.15, 0.05], gamma=0.9)
    assert keep.tolist() == [1, 1, 1, 0] and r == 3
    assert km >= np.float32(0.9) > pp
    # [0.4, 0.4, 0.2], gamma = 0.4 -> keep {0} (tie toward the lower index), tie reported
    keep, r, km, pp, tie = orc.keep_select([0.4, 0.4, 0.2], gamma=0.4)
    assert keep.tolist() == [1, 0, 0] and tie
    # gamma = 1 keeps every causal block, even zero-probability ones
    keep, r, *_ = orc.keep_select([1.0, 0.0, 0.0], gamma=1.0)
    assert keep.tolist() == [1, 1, 1]
    # non-causal blocks are never kept
    keep, *_ = orc.keep_select([0.5, 0.0, 0.5], causal_flags=[1, 0, 1], gamma=1.0)
    assert keep.tolist() == [1, 0, 1]


def test_keep_ratio_ranks_by_score_through_underflow(orc):
    # R9: keep-ratio keeps the top-k blocks by probability; the block softmax is monotone in S, so the
    # exact top-k is the top-k by score even where fp32 probabilities underflow to 0 (where ranking by
    # the rounded A would fall back to ascending j).  One head, one query block of 4 causal KV blocks.
    C, b = 128, 16
    S = np.full((1, 1, 4), -np.inf, np.float32)
    S[0, 0] = [20000.0, 0.0, 9000.0, 10.0]  # everything but block 0 underflows: t < -126
    out = orc.select(S, 1, b, 4 * b, C, b, select_mode=orc.SELECT_RATIO, keep_ratio=0.5)
    assert out["A"][0, 0, 1] == 0.0 and out["A"][0, 0, 2] == 0.0
    assert out["mass"][0, 0].tolist() == [1, 0, 1, 0]
    out = orc.select(S, 1, b, 4 * b, C, b, select_mode=orc.SELECT_RATIO, keep_ratio=0.75)
    assert out["mass"][0, 0].tolist() == [1, 0, 1, 1]


def test_keep_ratio(orc):
    A = np.array([0.1, 0.4, 0.2, 0.3], np.float32)
    keep, r, *_ = orc.keep_select(A, select=orc.SELECT_RATIO, keep_ratio=0.5)
    assert keep.tolist() == [0, 1, 0, 1] and r == 2
    keep, r, *_ = orc.keep_select(A, select=orc.SELECT_RATIO, keep_ratio=0.01)
    assert r == 1 and keep.tolist() == [0, 1, 0, 0]


@pytest.mark.parametrize("sigma", [0.05, 0.3, 1.0])
def test_select_invariants(orc, sigma):
    # mass >= gamma, minimality, monotone in gamma, OR over the head group, row 0
    rng = np.random.default_rng(int(sigma * 100))
    Hq, Hkv, N, C, b, g = 4, 2, 1024, 32, 64, 16
    q = (rng.standard_normal((Hq, N, C)) * sigma).astype(np.float32)
    k = (rng.standard_normal((Hkv, N, C)) * sigma).astype(np.float32)
    S = orc.block_scores(q, k, b, g)
    prev = None
    for gamma in [0.9, 0.95, 0.99, 0.999]:
        sel = orc.select(S, Hkv, N, N, C, b, gamma)
        mass, coarse = sel["mass"], sel["coarse"]
        A = sel["A"]
        kept = (A * mass).sum(-1, dtype=np.float64)
        assert (sel["kept_mass"] >= np.float32(gamma)).all()
        assert (sel["p_prev"] < np.float32(gamma)).all()
        # minimality: dropping the smallest kept block falls below gamma (ties exempt)
        for p in range(Hq):
            for i in range(S.shape[1]):
                kp = A[p, i][mass[p, i] == 1]
                assert kept[p, i] - kp.min() < gamma + 1e-5 or sel["tie"][p, i]
        assert np.array_equal(coarse, mass.reshape(Hkv, Hq // Hkv, *mass.shape[1:]).max(1))
        assert (mass[:, 0, 0] == 1).all()  # row 0 keeps block 0
        if prev is not None:
            assert ((prev == 1) <= (mass == 1)).all()  # monotone
        prev = mass
