"""Pins for the oracle's Stage 2 (Eq. 19-26): hash test vectors, closed-form densities,
degenerate configurations, statistical rates.  CPU only."""
import numpy as np
import pytest

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def test_mix64_splitmix_published_vectors(orc):
    # SplitMix64 (Steele, Lea & Flood, OOPSLA 2014; Vigna's splitmix64.c) seeded with 0 emits
    # mix64(k * golden) for k = 1, 2, 3: 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F.
    assert orc.mix64(GOLDEN) == 0xE220A8397B1DCDAF
    assert orc.mix64((2 * GOLDEN) & M64) == 0x6E789E6AA1B965F4
    assert orc.mix64((3 * GOLDEN) & M64) == 0x06C45D188009454F


def test_chi_psi_basic(orc):
    assert orc.chi(0, 0, 0) == orc.chi(0, 0, 0)
    assert orc.chi(0, 1, 0) != orc.chi(1, 0, 0)
    vals = [orc.psi(h, i, j, 7) for h in range(4) for i in range(64) for j in range(64)]
    assert all(0.0 <= x < 1.0 for x in vals)
    assert 0.45 <= np.mean(vals) <= 0.55


def test_chi_residues_uniform(orc):
    # over a 64x64 grid, residues mod 16 each appear with frequency 1/16 +- 0.05
    res = np.array([orc.chi(i, j, 0) % 16 for i in range(64) for j in range(64)])
    freq = np.bincount(res, minlength=16) / res.size
    assert np.all(np.abs(freq - 1 / 16) <= 0.05)
    # tighter: a chi-square-ish check (4096 draws, 16 bins) — each bin within 5 sigma
    sig = np.sqrt(4096 * (1 / 16) * (15 / 16))
    assert np.all(np.abs(np.bincount(res, minlength=16) - 256) <= 5 * sig)


def _causal_tiles(orc, Nq, Nkv, T):
    Tq, Tkv = -(-Nq // T), -(-Nkv // T)
    return np.array([[orc.causal(i, j, T, Nq, Nkv) for j in range(Tkv)] for i in range(Tq)])


def test_expand_identity_when_b_equals_T(orc):
    # b = T: tile mask = coarse mask restricted to tile causality
    rng = np.random.default_rng(0)
    N, T = 512, 64
    coarse = (rng.random((2, 8, 8)) < 0.3).astype(np.uint8)
    lab = orc.expand_rescue(coarse, N, N, T, T, n_sink=0, n_local=-1, eta=0, rho=0.0)
    cm = _causal_tiles(orc, N, N, T)
    assert np.array_equal(lab > 0, (coarse > 0) & cm[None])


def test_expand_4x4_patches(orc):
    # b = 256, T = 64: each kept coarse block -> a 4x4 tile patch (label mass)
    N = 1024
    coarse = np.zeros((1, 4, 4), np.uint8)
    coarse[0, 2, 1] = 1
    coarse[0, 3, 3] = 1
    lab = orc.expand_rescue(coarse, N, N, 256, 64, n_sink=0, n_local=-1, eta=0, rho=0.0)
    assert (lab[0, 8:12, 4:8] == orc.LBL_MASS).all()
    cm = _causal_tiles(orc, N, N, 64)
    diag = lab[0, 12:16, 12:16]
    assert np.array_equal(diag == orc.LBL_MASS, cm[12:16, 12:16])
    assert (lab > 0).sum() == 16 + cm[12:16, 12:16].sum()


def test_keep_all_is_full_causal(orc):
    # coarse full-causal -> tile mask = causal tile mask, density 1
    for Nq, Nkv in [(1000, 1000), (300, 1300), (64, 64), (65, 129)]:
        L, Lk = -(-Nq // 128), -(-Nkv // 128)
        coarse = np.ones((1, L, Lk), np.uint8)
        lab = orc.expand_rescue(coarse, Nq, Nkv, 128, 64, n_sink=0, n_local=-1, eta=0, rho=0.0)
        assert np.array_equal(lab[0] > 0, _causal_tiles(orc, Nq, Nkv, 64))


def test_band_and_sink(orc):
    N, T = 1024, 64
    L = N // T
    zero = np.zeros((1, N // 256, N // 256), np.uint8)
    cm = _causal_tiles(orc, N, N, T)
    # band saturation -> full causal
    lab = orc.expand_rescue(zero, N, N, 256, T, n_sink=1, n_local=L, eta=0, rho=0.0)
    assert np.array_equal(lab[0] > 0, cm)
    # n_local = 0 -> only the diagonal and column 0
    lab = orc.expand_rescue(zero, N, N, 256, T, n_sink=1, n_local=0, eta=0, rho=0.0)
    want = np.eye(L, dtype=bool) | (np.arange(L)[None, :] == 0)
    assert np.array_equal(lab[0] > 0, want)
    # sink + diagonal density on an L x L grid = (2L - 1) / (L (L + 1) / 2)
    assert (lab[0] > 0).sum() / cm.sum() == pytest.approx((2 * L - 1) / (L * (L + 1) / 2))
    assert (lab[0, :, 0] == orc.LBL_SINK).all()
    assert (np.diag(lab[0])[1:] == orc.LBL_BAND).all()
    # band of n_local + 1 tiles ending at the frontier, clipped at 0
    lab = orc.expand_rescue(zero, N, N, 256, T, n_sink=0, n_local=3, eta=0, rho=0.0)
    for i in range(L):
        assert np.nonzero(lab[0, i])[0].tolist() == list(range(max(0, i - 3), i + 1))


def test_band_chunked_frontier(orc):
    # chunked prefill (R18): Nq = 100, Nkv = 300, T = 64 -> d_0 = floor((200 + 63)/64) = 4
    zero = np.zeros((1, 1, 3), np.uint8)
    lab = orc.expand_rescue(zero, 100, 300, 128, 64, n_sink=0, n_local=1, eta=0, rho=0.0)
    assert np.nonzero(lab[0, 0])[0].tolist() == [3, 4]
    assert np.nonzero(lab[0, 1])[0].tolist() == [3, 4]  # d_1 = min(floor(327/64)=5, Tkv-1=4)


def test_label_precedence(orc):
    N = 512
    coarse = np.zeros((1, 2, 2), np.uint8)
    coarse[0, 1, 0] = 1  # mass block covering the sink column and part of the band
    lab = orc.expand_rescue(coarse, N, N, 256, 64, n_sink=1, n_local=8, eta=1, rho=1.0)
    assert lab[0, 4, 0] == orc.LBL_MASS  # mass beats sink
    assert lab[0, 1, 0] == orc.LBL_SINK  # sink beats band
    assert lab[0, 1, 1] == orc.LBL_BAND


def test_rescue_degenerate(orc):
    N = 2048
    cm = _causal_tiles(orc, N, N, 64)
    zero = np.zeros((1, 8, 8), np.uint8)
    # eta = 1 -> full causal
    lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=0, eta=1, rho=0.0)
    assert np.array_equal(lab[0] > 0, cm)
    # rho = 1 -> full causal
    lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=0, eta=0, rho=1.0)
    assert np.array_equal(lab[0] > 0, cm)
    # rho = 0, stride off -> no rescue labels
    lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=0, eta=0, rho=0.0)
    assert not np.isin(lab, [orc.LBL_STRIDE, orc.LBL_RANDOM]).any()


def test_rescue_rates(orc):
    # S:303 binomial +-3 sigma for rho; and the stride rule adds ~1/eta of the dropped tiles —
    # the paper's Tab.mask shows 8.75% -> 14.40% at eta = 16: 8.75 + 91.25/16 = 14.45.
    N = 8192
    zero = np.zeros((2, 32, 32), np.uint8)
    base = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=8, eta=0, rho=0.0)
    dropped = (~(base > 0)) & _causal_tiles(orc, N, N, 64)[None]
    nd = dropped.sum()
    for rho in [0.1, 0.3]:
        lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=8, eta=0, rho=rho)
        got = (lab == orc.LBL_RANDOM).sum()
        assert abs(got - rho * nd) <= 3 * np.sqrt(nd * rho * (1 - rho))
        assert ((lab > 0) >= (base > 0)).all()  # rescues only add tiles
    lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=8, eta=16, rho=0.0)
    got = (lab == orc.LBL_STRIDE).sum()
    assert abs(got - nd / 16) <= 3 * np.sqrt(nd / 16 * 15 / 16)
    # chi has no head index (R14): stride pattern identical across heads; psi differs
    assert np.array_equal(lab[0], lab[1])
    lab = orc.expand_rescue(zero, N, N, 256, 64, n_sink=1, n_local=8, eta=0, rho=0.3)
    assert not np.array_equal(lab[0], lab[1])
    # head_offset shifts psi's head index (multi-GPU shards must use global KV head ids)
    lab_off = orc.expand_rescue(zero[:1], N, N, 256, 64, n_sink=1, n_local=8, eta=0, rho=0.3, head_offset=1)
    assert np.array_equal(lab_off[0], lab[1])
