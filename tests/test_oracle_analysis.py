"""§8(f4): the paper's appendix error bound (Remark 1) and the Eq. 28-33 cost accounting, checked on
the oracle's masks (desk scale).  CPU only."""
import math

import numpy as np
import pytest


def _rand_case(rng, orc, N, T=32, m=2):
    q = rng.standard_normal((m, N, 16)).astype(np.float32)
    k = rng.standard_normal((1, N, 16)).astype(np.float32)
    v = rng.standard_normal((1, N, 16)).astype(np.float32)
    res = orc.mask_pipeline(q, k, b=64, g=16, T=T, gamma=float(rng.choice([0.5, 0.9, 0.99])),
                            n_local=int(rng.integers(0, 3)), eta=int(rng.choice([0, 4, 16])),
                            rho=float(rng.choice([0.0, 0.2])), seed=int(rng.integers(1 << 30)))
    return q, k, v, res["labels"]


def test_appendix_bound_holds_on_random_instances(orc):
    # holds on >= 200 random instances at N in {64, 128, 256}
    rng = np.random.default_rng(0)
    n = 0
    for N in [64, 128, 256]:
        for _ in range(70):
            q, k, v, lab = _rand_case(rng, orc, N)
            for r in orc.appendix_bound(q, k, v, lab, 32, 0.25):
                assert r["lhs"] <= r["rhs"] * (1 + 1e-9) + 1e-12
                n += 1
    assert n >= 200


def test_appendix_bound_zero_for_full_mask(orc):
    # full causal mask -> Z = Z_s, D = D_s, alpha = 0, lhs = 0
    rng = np.random.default_rng(1)
    q = rng.standard_normal((2, 96, 8)).astype(np.float32)
    k = rng.standard_normal((1, 96, 8)).astype(np.float32)
    v = rng.standard_normal((1, 96, 8)).astype(np.float32)
    lab = np.ones((1, 3, 3), np.uint8)
    for r in orc.appendix_bound(q, k, v, lab, 32, 0.3):
        assert r["alpha"] == 0.0 and r["lhs"] == 0.0


def test_mac_counts_match_closed_forms(orc):
    # Eq. 30: on full blocks stage-1 MACs = H_q sum_causal G^2 g C = H_q (L(L+1)/2) b^2 C / g;
    # Eq. 29: stage-2 MACs / dense MACs = kappa on full tiles; kappa = 1 -> dense count
    rng = np.random.default_rng(2)
    N, b, g, T, C, Hq = 512, 64, 16, 32, 16, 2
    q, k, v, lab = _rand_case(rng, orc, N, T=T, m=Hq)
    mc = orc.mac_counts(lab, N, N, C, Hq, b, g, T)
    L = N // b
    assert mc["stage1"] == Hq * (L * (L + 1) // 2) * (b // g) ** 2 * g * C
    assert mc["stage2"] / mc["dense"] == pytest.approx(mc["kappa"], abs=1e-12)
    Tq = N // T
    full = np.array([[[orc.causal(i, j, T, N, N) for j in range(Tq)] for i in range(Tq)]], np.uint8)
    mc1 = orc.mac_counts(full, N, N, C, Hq, b, g, T)
    assert mc1["stage2"] == mc1["dense"] and mc1["kappa"] == 1.0
    # dense MACs of causal tiles incl. the diagonal = 2 C m T^2 Tq(Tq+1)/2 on full tiles
    assert mc1["dense"] == 2 * C * Hq * T * T * Tq * (Tq + 1) // 2
