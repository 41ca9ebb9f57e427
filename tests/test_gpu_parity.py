"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Masks (coarse bits, tile labels, lists, counts) must be bit-exact; O within max-abs 2e-2 and
mean-abs 2e-3 of the fp64 oracle (BASELINE.json).  Sizes span several tiles and ragged tails."""
import ctypes
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import paper_2605_12193_b200 as bf
import workloads
from gpu_util import check_lists, compare_o, f32, oracle_attention, oracle_masks, run_gpu

pytestmark = pytest.mark.gpu

TINY = dict(B=1, Hq=2, Hkv=1, Nq=2048, Nkv=2048, d=128)
TINY_CFG = dict(b=128, g=64, T=64)


def _check_masks(gpu, ref, cfg):
    coarse = np.stack([x["coarse"] for x in ref])
    labels = np.stack([x["labels"] for x in ref])
    assert np.array_equal(gpu["coarse"], coarse), "coarse mask mismatch"
    assert np.array_equal(gpu["labels"], labels), "tile label mismatch"
    assert np.array_equal(gpu["tiles"], (labels > 0).astype(np.uint8)), "tile bits mismatch"
    if gpu.get("kept_mass") is not None:
        km = np.stack([x["kept_mass"] for x in ref])
        assert np.array_equal(gpu["kept_mass"], km), "kept mass mismatch"
    ties = sum(int(x["tie"].sum()) for x in ref)
    assert gpu["stats"]["rows_exact_tie"] == ties
    assert gpu["stats"]["kept_tiles"] == int((labels > 0).sum())
    return labels


@pytest.mark.parametrize("sigma,seed", [(1.0, 1), (0.7, 2), (0.5, 3), (0.3, 4)])
@pytest.mark.parametrize("gamma", [0.9, 0.99, 0.999])
def test_tiny_gaussian_masks_and_output(sigma, seed, gamma):
    prob = workloads.gaussian(seed, **TINY, sigma=sigma)
    cfg = bf.Config(**TINY_CFG, gamma=gamma)
    gpu = run_gpu(prob, cfg)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    check_lists(gpu, labels, 2048, 2048, 64)
    (o_ref, lse_ref), = oracle_attention(prob, labels, 64)
    compare_o(gpu["o"][0], o_ref, f"sigma={sigma} gamma={gamma}")
    lse = gpu["lse"][0].cpu().numpy()
    assert np.abs(lse - lse_ref).max() <= 1e-3


def test_tiny_structured():
    prob = workloads.structured(101, **TINY, block=128)
    cfg = bf.Config(**TINY_CFG)
    gpu = run_gpu(prob, cfg)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    (o_ref, _), = oracle_attention(prob, labels, 64)
    compare_o(gpu["o"][0], o_ref, "structured")


@pytest.mark.parametrize("case", [
    dict(B=2, Hq=4, Hkv=1, Nq=1000, Nkv=1000, b=128, g=64),      # ragged tail, m=4 (NQT=2)
    dict(B=1, Hq=8, Hkv=1, Nq=777, Nkv=1500, b=256, g=64),       # chunked prefill, m=8 (2 chunks)
    dict(B=1, Hq=3, Hkv=3, Nq=640, Nkv=640, b=64, g=16),         # m=1 (half-empty Q tile)
    dict(B=1, Hq=4, Hkv=2, Nq=130, Nkv=4000, b=256, g=32),       # long context, short chunk, G=8
    dict(B=1, Hq=2, Hkv=1, Nq=1, Nkv=1, b=64, g=64),             # single token
    dict(B=1, Hq=16, Hkv=2, Nq=520, Nkv=520, b=128, g=128),      # G=1, m=8
])
def test_shapes(case):
    c = dict(case)
    b, g = c.pop("b"), c.pop("g")
    prob = workloads.gaussian(11, d=128, sigma=0.8, **c)
    cfg = bf.Config(b=b, g=g, T=64, gamma=0.95, eta=4, rho=0.2, seed=5)
    gpu = run_gpu(prob, cfg)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    check_lists(gpu, labels, c["Nq"], c["Nkv"], 64)
    # ragged tails run the tensor-core scores over full groups + the canonical partial-group fixup
    # (AUTO); the all-canonical SIMT path must give the same bits
    canon = run_gpu(prob, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), lse=False)
    assert np.array_equal(canon["coarse"], gpu["coarse"]) and np.array_equal(canon["labels"], gpu["labels"])
    for r, (o_ref, lse_ref) in enumerate(oracle_attention(prob, labels, 64)):
        compare_o(gpu["o"][r], o_ref, str(case))
        assert np.abs(gpu["lse"][r].cpu().numpy() - lse_ref).max() <= 1e-3


def test_kept_mass_canonical():
    prob = workloads.gaussian(5, **TINY, sigma=0.6)
    cfg = bf.Config(**TINY_CFG, gamma=0.95)
    gpu = run_gpu(prob, cfg, kept_mass=True)
    _check_masks(gpu, oracle_masks(prob, cfg), cfg)


@pytest.mark.parametrize("dist", ["g1.0", "g0.5", "g0.2", "structured"])
@pytest.mark.parametrize("gamma", [0.9, 0.99])
def test_fast_scores_certified_equal_canonical(dist, gamma):
    """AUTO (tcgen05 + certification + canonical recompute) and CANONICAL give the same mask,
    equal to the oracle's; the observed tensor-core score error sits far below tau."""
    shape = dict(B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128)
    if dist == "structured":
        prob = workloads.structured(7, **shape, block=256)
    else:
        prob = workloads.gaussian(8, **shape, sigma=float(dist[1:]))
    fast = run_gpu(prob, bf.Config(b=256, g=64, gamma=gamma, scores=bf.SCORES_AUTO))
    canon = run_gpu(prob, bf.Config(b=256, g=64, gamma=gamma, scores=bf.SCORES_CANONICAL))
    assert np.array_equal(fast["coarse"], canon["coarse"])
    assert np.array_equal(fast["labels"], canon["labels"])
    assert torch.equal(fast["o"], canon["o"])
    ref = oracle_masks(prob, bf.Config(b=256, g=64, gamma=gamma))
    _check_masks(fast, ref, None)
    st = fast["stats"]
    print(f"{dist} gamma={gamma}: flagged head rows {st['rows_flagged']} / {st['rows']}, "
          f"groups recomputed {st['rows_recomputed']}")
    # tensor-core scores (workspace head) vs oracle canonical scores on certified rows, relative to
    # ||x|| ||y|| bounds: must stay far below tau (api.cu certify_tau)
    Lq = Lkv = 16
    S_fast = fast["ws"][: 8 * Lq * Lkv * 4].view(torch.float32).view(8, Lq, Lkv).cpu().numpy()
    S_can = ref[0]["S"]
    qf = f32(prob.q[0]).reshape(8, Lq, 4, 64 * 128)
    kf = f32(prob.k[0]).reshape(2, Lkv, 4, 64 * 128)
    qn = np.linalg.norm(qf.astype(np.float64), axis=-1).max(-1)
    kn = np.linalg.norm(kf.astype(np.float64), axis=-1).max(-1)
    bound = qn[:, :, None] * np.repeat(kn, 4, axis=0)[:, None, :]
    tri = np.tril(np.ones((Lq, Lkv), bool))
    ratio = (np.abs(S_fast - S_can) / bound)[:, tri].max()
    n, u = 64 * 128, 2.0 ** -24
    # api.cu certify_tau: worst-case canonical term gamma_{C+g} plus the tensor-core chain (2 n/16 u);
    # 2 u per split-K partial is not counted here (it only makes tau larger)
    tau = (128 + 64) * u / (1 - (128 + 64) * u) + u * n / 8
    print(f"max |S_tc - S_canon| / (|x||y|) = {ratio:.3e}  (tau = {tau:.3e}, ratio {ratio / tau:.3f})")
    # the bound is a worst case (every rounding of both orders aligned); on these inputs the
    # observed difference must sit at most a quarter of it, so the certification has >= 4x headroom
    assert ratio < tau / 4


def _ws_norms(ws: torch.Tensor, B, Hq, Hkv, Nq, Nkv, d, b, T=64, paged=False):
    """qn / kn from the workspace (layout of api.cu ws_layout, 256-byte aligned segments)."""
    al = lambda x: (x + 255) & ~255
    cd = lambda a, c: -(-a // c)
    Lq, Lkv, Tq, Tkv = cd(Nq, b), cd(Nkv, b), cd(Nq, T), cd(Nkv, T)
    a = Nc = Nkv - Nq
    a = cd(Nc, T) + 1
    i0 = max(Tkv - a, 0)
    causal = (i0 * a + i0 * (i0 - 1) // 2 + (Tq - i0) * Tkv) if Tq > i0 else (Tq * a + Tq * (Tq - 1) // 2)
    o = 0
    for size in [B * Hq * Lq * Lkv * 4, B * Hq * Lq * d * 4, B * Hkv * Lkv * d * 4, B * Hkv * Lq * cd(Lkv, 32) * 4,
                 B * Hkv * Tq * cd(Tkv, 32) * 4, B * Hkv * causal * 4, B * Hkv * Tq * 4]:
        o += al(size)
    o += al(ctypes.sizeof(bf.bfla_stats))
    qn = ws[o:o + B * Hq * Lq * 4].view(torch.float32).view(B, Hq, Lq).cpu().numpy()
    o += al(B * Hq * Lq * 4)
    kn = ws[o:o + B * Hkv * Lkv * 4].view(torch.float32).view(B, Hkv, Lkv).cpu().numpy()
    return qn, kn


@pytest.mark.parametrize("m", [1, 2, 4, 8])
def test_certification_norms(m):
    """The certification bounds of the fast Stage-1 path (block maxima of the group l2 norms, DESIGN.md
    §4) bound the exact norms from above and stay within 2^-9 of them, for G = 4 groups per block and
    every GQA group size; AUTO masks equal CANONICAL masks.  N = 20480 gives two score N tiles."""
    B, Hkv, N, d, b = 1, 2, 20480, 128, 256
    Hq = m * Hkv
    prob = workloads.gaussian(31 + m, B=B, Hq=Hq, Hkv=Hkv, Nq=N, Nkv=N, d=d, sigma=0.8)
    fast = run_gpu(prob, bf.Config(b=b, g=64, gamma=0.95, scores=bf.SCORES_AUTO), lse=False)
    canon = run_gpu(prob, bf.Config(b=b, g=64, gamma=0.95, scores=bf.SCORES_CANONICAL), lse=False)
    assert np.array_equal(fast["coarse"], canon["coarse"])
    assert np.array_equal(fast["labels"], canon["labels"])
    qn, kn = _ws_norms(fast["ws"], B, Hq, Hkv, N, N, d, b)
    L = N // b
    qx = prob.q[0].float().reshape(Hq, L, b // 64, 64 * d).norm(dim=-1).amax(-1).double().numpy()
    kx = prob.k[0].float().reshape(Hkv, L, b // 64, 64 * d).norm(dim=-1).amax(-1).double().numpy()
    # both kernels round the fp32 norm up by exactly (1 + 2^-10); their fp32 sums are within 2^-14 of
    # the exact norm, so the ratio pins the whole sum (a dropped or doubled k-step moves it by ~2^-8)
    for got, want in ((qn[0], qx), (kn[0], kx)):
        r = got / want
        assert (r >= (1 + 2 ** -10) * (1 - 2 ** -14)).all(), ("norm bound low", r.min())
        assert (r <= (1 + 2 ** -10) * (1 + 2 ** -14)).all(), ("norm bound loose", r.max())


@pytest.mark.parametrize("T", [64, 128])
@pytest.mark.parametrize("case", [
    dict(Nq=1000, Nkv=1500, b=128, paged=0),      # chunked, ragged: canonical SIMT scores
    dict(Nq=2048, Nkv=2048, b=256, paged=0),      # tensor-core scores + certification + recompute
    dict(Nq=2048, Nkv=2048, b=256, paged=16),     # paged K/V
])
def test_per_query_head_masks(case, T):
    """§8 f3: BFLA_MASK_PER_Q_HEAD keeps Eq. 18 literal (one mask per query head, Stage 2 per query
    head, psi by query head).  Reference: the oracle on K/V repeated per query head, where the OR over
    a one-head group is that head's own mask; masks bit-exact, O within tolerance."""
    m = 4
    prob = workloads.gaussian(41, B=1, Hq=8, Hkv=2, Nq=case["Nq"], Nkv=case["Nkv"], d=128, sigma=0.8)
    if case["b"] % T:
        pytest.skip("T must divide b")
    cfg = bf.Config(b=case["b"], g=64, T=T, gamma=0.95, eta=4, rho=0.2, seed=5, mask_groups=bf.MASK_PER_Q_HEAD)
    gpu = run_gpu(prob, cfg, paged_page=case["paged"])
    rep = workloads.Problem(q=prob.q, k=prob.k.repeat_interleave(m, dim=1), v=prob.v.repeat_interleave(m, dim=1))
    ref = oracle_masks(rep, cfg)
    labels = _check_masks(gpu, ref, cfg)
    assert labels.shape[1] == 8
    check_lists(gpu, labels, case["Nq"], case["Nkv"], T)
    (o_ref, lse_ref), = oracle_attention(rep, labels, T)
    compare_o(gpu["o"][0], o_ref, str(case))
    assert np.abs(gpu["lse"][0].cpu().numpy() - lse_ref).max() <= 1e-3


@pytest.mark.parametrize("case", [
    dict(B=2, Hq=8, Hkv=2, Nq=1000, Nkv=1000, d=128, b=256, g=64, paged=0),   # m=4: 2 chunks of 1 head x 128 rows
    dict(B=1, Hq=8, Hkv=1, Nq=700, Nkv=1500, d=128, b=256, g=64, paged=16),   # chunked prefill, paged, m=8
    dict(B=1, Hq=2, Hkv=2, Nq=1111, Nkv=1111, d=128, b=128, g=64, paged=0),   # m=1, T = b
    dict(B=1, Hq=4, Hkv=2, Nq=900, Nkv=900, d=256, b=256, g=64, paged=0),     # d=256 kernel
])
def test_tile_128(case):
    """T = 128 mask tiles: Stage 2 at T = 128 and the prefill kernels, which run
    each kept 128-key tile as two 64-key halves and 128-row Q tiles of one head; bit-exact masks and O
    within tolerance against the oracle at the same T, ragged tails included."""
    c = dict(case)
    b, g, d, paged = c.pop("b"), c.pop("g"), c.pop("d"), c.pop("paged")
    prob = workloads.gaussian(21, d=d, sigma=0.8, **c)
    cfg = bf.Config(b=b, g=g, T=128, gamma=0.95, eta=4, rho=0.2, seed=7)
    gpu = run_gpu(prob, cfg, paged_page=paged)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    check_lists(gpu, labels, c["Nq"], c["Nkv"], 128)
    for r, (o_ref, lse_ref) in enumerate(oracle_attention(prob, labels, 128)):
        compare_o(gpu["o"][r], o_ref, str(case))
        assert np.abs(gpu["lse"][r].cpu().numpy() - lse_ref).max() <= 1e-3


@pytest.mark.parametrize("ratio", [0.05, 0.2, 0.6])
def test_keep_ratio_fast_path(ratio):
    """Keep-ratio (R9, ranked by score) on the tensor-core path: certification by the score gap at the
    cut, recompute of the cut's neighbourhood only; AUTO == CANONICAL == oracle, bit for bit."""
    prob = workloads.structured(9, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128, block=256)
    kw = dict(b=256, g=64, select=bf.SELECT_RATIO, keep_ratio=ratio)
    fast = run_gpu(prob, bf.Config(**kw, scores=bf.SCORES_AUTO), lse=False)
    canon = run_gpu(prob, bf.Config(**kw, scores=bf.SCORES_CANONICAL), lse=False)
    assert np.array_equal(fast["coarse"], canon["coarse"])
    assert np.array_equal(fast["labels"], canon["labels"])
    _check_masks(fast, oracle_masks(prob, bf.Config(**kw)), None)
    print(f"ratio {ratio}: flagged {fast['stats']['rows_flagged']} of {fast['stats']['rows']}")


@pytest.mark.parametrize("d", [128, 256])
@pytest.mark.parametrize("ratio", [0.05, 0.3])
def test_keep_ratio_recompute_band(ratio, d):
    """Keep-ratio rows that fail certification recompute only the blocks whose fast score lies in the
    band s_cut -/+ 2d around the cut (stage1_select.cu): outside it the rank against the canonical
    k-th score is already certain.  A widened error bound (bfla_config.certify_slack) flags most rows and
    widens every band, so rows mix fast and canonical scores; the mask must still equal the oracle's bit
    for bit (d = 128: TMA recompute kernel; d = 256: the chunked TMA one)."""
    prob = workloads.structured(10, B=1, Hq=4, Hkv=2, Nq=3072, Nkv=3072, d=d, block=256)
    kw = dict(b=256, g=64, select=bf.SELECT_RATIO, keep_ratio=ratio)
    fast = run_gpu(prob, bf.Config(**kw, scores=bf.SCORES_AUTO, certify_slack=3000.0), lse=False)
    assert fast["stats"]["rows_flagged"] >= 8, fast["stats"]
    _check_masks(fast, oracle_masks(prob, bf.Config(**kw)), None)


@pytest.mark.parametrize("paged", [0, 16])
def test_dynamic_and_static_item_order_identical(paged):
    """The prefill kernels take their work items from a workspace counter when a workspace is given
    (greedy longest-first scheduling) and round-robin without one: every item is computed the same
    way whichever CTA takes it, so O and LSE are bitwise identical (sparse and dense)."""
    prob = workloads.structured(12, B=2, Hq=8, Hkv=2, Nq=3000, Nkv=3000, d=128, block=256)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    if paged:
        kc, vc, pt = workloads.paged(k, v, paged, seed=4, extra_pages=3)
    outs = []
    for use_ws in (True, False):
        o = torch.empty_like(q)
        l = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
        P = (bf.make_problem(q, kc, vc, o, l, page_table=pt, n_kv=k.shape[2]) if paged
             else bf.make_problem(q, k, v, o, l))
        cfg = bf.Config(b=256, g=64)
        ws = bf.alloc_workspace(P, cfg)
        m = bf.alloc_mask(P, cfg)
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill(P, cfg, m, ws if use_ws else None)
        od = torch.empty_like(q)
        Pd = (bf.make_problem(q, kc, vc, od, page_table=pt, n_kv=k.shape[2]) if paged
              else bf.make_problem(q, k, v, od))
        bf.bfla_prefill(Pd, None, None, bf.alloc_workspace(Pd, None) if use_ws else None)
        torch.cuda.synchronize()
        outs.append((o.clone(), l.clone(), od.clone()))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_whole_path_deterministic():
    """S:513 / §8(b): identical inputs give identical bits — masks, lists, O and LSE of two runs of the
    whole path (tensor-core Stage 1 with certification and recompute, dynamic item scheduling)."""
    prob = workloads.structured(13, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128, block=256)
    cfg = bf.Config(b=256, g=64, eta=8, rho=0.1, seed=3)
    a, b = run_gpu(prob, cfg), run_gpu(prob, cfg)
    for key in ("coarse", "tiles", "labels", "count", "list"):
        assert np.array_equal(a[key], b[key]), key
    assert torch.equal(a["o"], b["o"]) and torch.equal(a["lse"], b["lse"])


def test_mean_pool_and_keep_ratio():
    prob = workloads.gaussian(21, B=1, Hq=4, Hkv=2, Nq=1500, Nkv=1500, d=128, sigma=1.0)
    for cfg in [bf.Config(b=128, g=64, pool=bf.POOL_MEAN, gamma=0.9),
                bf.Config(b=128, g=64, select=bf.SELECT_RATIO, keep_ratio=0.2),
                bf.Config(b=128, g=64, pool=bf.POOL_MEAN, select=bf.SELECT_RATIO, keep_ratio=0.05)]:
        gpu = run_gpu(prob, cfg)
        ref = oracle_masks(prob, cfg)
        labels = _check_masks(gpu, ref, cfg)
        (o_ref, _), = oracle_attention(prob, labels, 64)
        compare_o(gpu["o"][0], o_ref, str(cfg))


def test_stage2_isolated_rescue_variants():
    """Stage 2 alone: upload an arbitrary coarse mask, compare labels/lists with the oracle."""
    rng = np.random.default_rng(3)
    B, Hkv, N = 2, 3, 3000
    prob = workloads.gaussian(1, B=B, Hq=Hkv * 2, Hkv=Hkv, Nq=N, Nkv=N, d=128)
    for kw in [dict(n_sink=1, n_local=8, eta=16, rho=0.0), dict(n_sink=2, n_local=0, eta=0, rho=0.3, seed=99),
               dict(n_sink=0, n_local=3, eta=1, rho=0.0), dict(n_sink=1, n_local=2, eta=7, rho=0.5, seed=1 << 40)]:
        cfg = bf.Config(b=256, g=64, **kw)
        q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
        o = torch.empty_like(q)
        P = bf.make_problem(q, k, v, o, head_offset=5)
        m = bf.alloc_mask(P, cfg, labels=True)
        coarse = (rng.random((B, Hkv, m.Lq, m.Lkv)) < 0.1).astype(np.uint8)
        words = np.zeros(m.coarse_bits.shape, np.int64)
        for j in range(m.Lkv):
            words[..., j // 32] |= coarse[..., j].astype(np.int64) << (j % 32)
        words = np.where(words >= 2 ** 31, words - 2 ** 32, words)
        m.coarse_bits.copy_(torch.from_numpy(words.astype(np.int32)))
        bf.bfla_expand_rescue(P, cfg, m)
        torch.cuda.synchronize()
        want = np.stack([oracle.expand_rescue(coarse[r], N, N, 256, 64, cfg.n_sink, cfg.n_local, cfg.eta, cfg.rho,
                                              cfg.seed, head_offset=5) for r in range(B)])
        assert np.array_equal(m.tile_label.cpu().numpy(), want)
        gpu = dict(count=m.tile_count.cpu().numpy(), list=m.tile_list.cpu().numpy())
        check_lists(gpu, want, N, N, 64)


def test_dense_matches_oracle_and_sdpa():
    prob = workloads.gaussian(31, B=1, Hq=4, Hkv=2, Nq=1100, Nkv=1300, d=128, sigma=1.0)
    gpu = run_gpu(prob, None)
    (o_ref, lse_ref), = oracle_attention(prob, None, 64)
    compare_o(gpu["o"][0], o_ref, "dense")
    assert np.abs(gpu["lse"][0].cpu().numpy() - lse_ref).max() <= 1e-3


def test_keep_all_sparse_equals_dense_bitwise():
    prob = workloads.gaussian(41, B=1, Hq=8, Hkv=2, Nq=1280, Nkv=1280, d=128, sigma=0.5)
    dense = run_gpu(prob, None)
    sparse = run_gpu(prob, bf.Config(b=128, g=64, gamma=1.0))
    assert torch.equal(dense["o"], sparse["o"])
    assert torch.equal(dense["lse"], sparse["lse"])


@pytest.mark.parametrize("page", [16, 32, 64])
def test_paged_equals_contiguous(page):
    prob = workloads.gaussian(51, B=2, Hq=8, Hkv=2, Nq=1000, Nkv=1000, d=128, sigma=0.9)
    cfg = bf.Config(b=128, g=64, gamma=0.95, eta=8, rho=0.1)
    a = run_gpu(prob, cfg)
    b = run_gpu(prob, cfg, paged_page=page)
    assert np.array_equal(a["labels"], b["labels"])
    assert torch.equal(a["o"], b["o"]), "paged O differs from contiguous O"
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(b, ref, cfg)
    for r, (o_ref, _) in enumerate(oracle_attention(prob, labels, 64)):
        compare_o(b["o"][r], o_ref, f"paged {page}")


def test_head_dim_256():
    prob = workloads.gaussian(61, B=1, Hq=4, Hkv=2, Nq=900, Nkv=900, d=256, sigma=0.8)
    cfg = bf.Config(b=128, g=64, gamma=0.95)
    gpu = run_gpu(prob, cfg)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    (o_ref, _), = oracle_attention(prob, labels, 64)
    compare_o(gpu["o"][0], o_ref, "d=256")
    dense = run_gpu(prob, None)
    (o_ref, _), = oracle_attention(prob, None, 64)
    compare_o(dense["o"][0], o_ref, "d=256 dense")


def test_strided_views_and_batch():
    # q/o as strided views of a [B, N, H, d] buffer (token-major, like a fused QKV projection)
    B, Hq, Hkv, N, d = 2, 4, 2, 700, 128
    prob = workloads.gaussian(71, B=B, Hq=Hq, Hkv=Hkv, Nq=N, Nkv=N, d=d)
    qt = prob.q.cuda().transpose(1, 2).contiguous().transpose(1, 2)  # strides (N*H*d, d, H*d, 1)
    ot = torch.empty(B, N, Hq, d, dtype=torch.bfloat16, device="cuda").transpose(1, 2)
    cfg = bf.Config(b=128, g=64)
    P = bf.make_problem(qt, prob.k.cuda(), prob.v.cuda(), ot)
    bf.bfla_prefill(P, cfg, None, bf.alloc_workspace(P, cfg))
    ref = run_gpu(prob, cfg)
    assert torch.equal(ot.contiguous(), ref["o"])


def _varlen_case(seed, lens, Hq=4, Hkv=2, d=128):
    """Padded varlen batch: request r uses q[r, :, :n_q_r], k/v[r, :, :n_kv_r]; the padding holds
    large garbage that must not reach any result."""
    B = len(lens)
    Nq, Nkv = max(a for a, _ in lens), max(b for _, b in lens)
    prob = workloads.gaussian(seed, B, Hq, Hkv, Nq, Nkv, d, sigma=0.8)
    q, k, v = prob.q.clone(), prob.k.clone(), prob.v.clone()
    for r, (nq, nkv) in enumerate(lens):
        q[r, :, nq:] = 1e4
        k[r, :, nkv:] = -1e4
        v[r, :, nkv:] = 1e4
    return workloads.Problem(q, k, v), torch.tensor(lens, dtype=torch.int32)


@pytest.mark.parametrize("T", [64, 128])
@pytest.mark.parametrize("paged", [0, 16])
def test_varlen_batch(paged, T):
    lens = [(700, 1500), (300, 300), (129, 1000), (64, 64)]
    prob, sl = _varlen_case(81, lens)
    cfg = bf.Config(b=128, g=64, T=T, gamma=0.95, eta=4, rho=0.2, seed=3)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    B, Hq, Nq, d = q.shape
    Nkv = k.shape[2]
    o = torch.zeros_like(q)
    l = torch.zeros(B, Hq, Nq, dtype=torch.float32, device="cuda")
    if paged:
        kc, vc, pt = workloads.paged(k, v, paged, seed=5, extra_pages=2)
        P = bf.make_problem(q, kc, vc, o, l, page_table=pt, n_kv=Nkv, seqlens=sl)
    else:
        P = bf.make_problem(q, k, v, o, l, seqlens=sl)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg, labels=True)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    torch.cuda.synchronize()
    # varlen Stage 1 runs on the tensor cores (full groups) + the canonical partial-group fixup; the
    # all-canonical path gives the same coarse mask
    mc = bf.alloc_mask(P, cfg)
    bf.bfla_block_mask(P, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), mc, bf.alloc_workspace(P, cfg))
    torch.cuda.synchronize()
    assert torch.equal(mc.coarse_bits, m.coarse_bits)
    coarse, labels = m.coarse_dense().cpu().numpy(), m.tile_label.cpu().numpy()
    counts, lists = m.tile_count.cpu().numpy(), m.tile_list.cpu().numpy()
    Tq_max, Tkv_max = labels.shape[2], labels.shape[3]
    for r, (nq, nkv) in enumerate(lens):
        qf, kf, vf = (f32(t[r])[:, :n] for t, n in ((prob.q, nq), (prob.k, nkv), (prob.v, nkv)))
        ref = oracle.mask_pipeline(qf, kf, b=128, g=64, T=T, gamma=0.95, eta=4, rho=0.2, seed=3)
        Lq, Lkv = ref["coarse"].shape[1:]
        assert np.array_equal(coarse[r, :, :Lq, :Lkv], ref["coarse"]), r
        assert not coarse[r, :, Lq:].any() and not coarse[r, :, :, Lkv:].any()
        Tq, Tkv = ref["labels"].shape[1:]
        assert np.array_equal(labels[r, :, :Tq, :Tkv], ref["labels"]), r
        assert not labels[r, :, Tq:].any() and not labels[r, :, :, Tkv:].any()
        # lists: row (r, h, i) at (r*Hkv + h) * Tq_max*Tkv_max + causal prefix of request r
        rc = np.array([sum(oracle.causal(i, j, T, nq, nkv) for j in range(Tkv)) for i in range(Tq)])
        offs = np.concatenate([[0], np.cumsum(rc)])
        for h in range(2):
            for i in range(Tq):
                want = np.nonzero(ref["labels"][h, i])[0]
                base = (r * 2 + h) * Tq_max * Tkv_max + offs[i]
                assert counts[r, h, i] == len(want)
                assert np.array_equal(lists[base:base + len(want)], want)
            assert not counts[r, h, Tq:].any()
        O_ref, lse_ref = oracle.masked_attention(qf, kf, vf, 128 ** -0.5, ref["labels"], T)
        compare_o(o[r, :, :nq], O_ref, f"varlen r={r}")
        assert np.abs(l[r, :, :nq].cpu().numpy() - lse_ref).max() <= 1e-3
        assert not o[r, :, nq:].float().abs().sum().item()  # padding rows untouched (zeros)


def test_varlen_dense_and_single_call():
    lens = [(500, 900), (256, 256), (77, 333)]
    prob, sl = _varlen_case(82, lens, Hq=8, Hkv=2)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o = torch.zeros_like(q)
    bf.bfla_prefill(bf.make_problem(q, k, v, o, seqlens=sl), None, None, None)  # dense causal
    cfg = bf.Config(b=128, g=64, gamma=1.0)  # keep-all through the whole sparse path
    o2 = torch.zeros_like(q)
    P2 = bf.make_problem(q, k, v, o2, seqlens=sl)
    bf.bfla_prefill(P2, cfg, None, bf.alloc_workspace(P2, cfg))
    torch.cuda.synchronize()
    assert torch.equal(o, o2)
    for r, (nq, nkv) in enumerate(lens):
        qf, kf, vf = (f32(t[r])[:, :n] for t, n in ((prob.q, nq), (prob.k, nkv), (prob.v, nkv)))
        O_ref, _ = oracle.masked_attention(qf, kf, vf, 128 ** -0.5)
        compare_o(o[r, :, :nq], O_ref, f"varlen dense r={r}")


def _lpt_rows(rho0, rho1, B, H, Tq):
    """(r, h, i) of the LPT-order rows [rho0, rho1) (include/bfla.h, bfla_sparse_prefill_rows)."""
    out = []
    for rho in range(rho0, rho1):
        seg, i = divmod(rho, Tq)
        out.append((seg // H, seg % H, Tq - 1 - i))
    return out


@pytest.mark.parametrize("case", [
    dict(B=2, Hq=8, Hkv=2, N=3000, d=128, paged=0),     # m=4 (NQT=2), two requests
    dict(B=1, Hq=8, Hkv=2, N=3000, d=128, paged=16),    # paged K/V
    dict(B=1, Hq=16, Hkv=2, N=2500, d=128, paged=0),    # m=8: two head chunks per row
    dict(B=1, Hq=4, Hkv=2, N=2000, d=256, paged=0),     # d=256 kernel
])
def test_row_slices_compose_to_full_prefill(case):
    """§8 f2: slicing the prefill by LPT rows (bfla_sparse_prefill_rows) over a cost-balanced partition
    (bfla_balance_rows) reproduces the unsliced O and LSE bit for bit, and one slice writes exactly its
    rows' (heads, tokens) and nothing else."""
    B, Hq, Hkv, N, d, paged = (case[k] for k in ("B", "Hq", "Hkv", "N", "d", "paged"))
    prob = workloads.structured(14, B=B, Hq=Hq, Hkv=Hkv, Nq=N, Nkv=N, d=d, block=256)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    if paged:
        kc, vc, pt = workloads.paged(k, v, paged, seed=6, extra_pages=2)

    def problem(o, l):
        return (bf.make_problem(q, kc, vc, o, l, page_table=pt, n_kv=N) if paged
                else bf.make_problem(q, k, v, o, l))

    cfg = bf.Config(b=256, g=64, eta=8, rho=0.1, seed=9)
    o_full = torch.empty_like(q)
    l_full = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    P = problem(o_full, l_full)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    counts = m.tile_count.view(B, Hkv, -1).cpu()
    Tq = counts.shape[2]
    bounds = bf.bfla_balance_rows(counts, 3)
    assert bounds[0] == 0 and bounds[-1] == B * Hkv * Tq

    sentinel_o, sentinel_l = 7.0, -5.0
    o_s = torch.full_like(q, sentinel_o)
    l_s = torch.full(q.shape[:3], sentinel_l, dtype=torch.float32, device="cuda")
    Ps = problem(o_s, l_s)
    for a, b_ in zip(bounds[:-1], bounds[1:]):
        bf.bfla_sparse_prefill_rows(Ps, cfg, m, a, b_, ws)
    torch.cuda.synchronize()
    assert torch.equal(o_s, o_full) and torch.equal(l_s, l_full)
    # the composed slices against the CPU oracle itself (masks from the oracle, fp64 Eq. 27): every
    # slice boundary row plus a sample of the rest, all heads
    ref = oracle_masks(prob, cfg)
    labels = np.stack([x["labels"] for x in ref])
    assert np.array_equal(m.tile_dense().cpu().numpy(), (labels > 0).astype(np.uint8))
    rows_t = sorted({min(N - 1, i * 64 + off) for i in range(0, -(-N // 64), 5) for off in (0, 63)}
                    | {min(N - 1, (Tq - 1 - (bb % Tq)) * 64) for bb in bounds[1:-1]})
    for r in range(B):
        rows = np.array([[p_, t] for p_ in range(Hq) for t in rows_t], np.int32)
        (o_ref, lse_ref), = oracle_attention(workloads.Problem(prob.q[r:r + 1], prob.k[r:r + 1], prob.v[r:r + 1]),
                                             labels[r:r + 1], 64, rows_per_req=[rows])
        og = o_s[r].float().cpu().numpy()[rows[:, 0], rows[:, 1]].astype(np.float64)
        err = np.abs(og - o_ref)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
        assert np.abs(l_s[r].cpu().numpy()[rows[:, 0], rows[:, 1]] - lse_ref).max() <= 1e-3

    # one slice alone: exactly its rows
    a, b_ = bounds[1], bounds[2]
    o_1 = torch.full_like(q, sentinel_o)
    l_1 = torch.full(q.shape[:3], sentinel_l, dtype=torch.float32, device="cuda")
    bf.bfla_sparse_prefill_rows(problem(o_1, l_1), cfg, m, a, b_, None)
    torch.cuda.synchronize()
    want = torch.zeros(q.shape[:3], dtype=torch.bool)
    mh = Hq // Hkv
    for r, h, i in _lpt_rows(a, b_, B, Hkv, Tq):
        want[r, h * mh:(h + 1) * mh, i * 64:(i + 1) * 64] = True
    want = want.cuda()
    assert torch.equal(o_1[want], o_full[want]) and torch.equal(l_1[want], l_full[want])
    assert bool((o_1[~want] == sentinel_o).all()) and bool((l_1[~want] == sentinel_l).all())
    # empty slices enqueue nothing; out-of-range slices are rejected before any launch
    bf.bfla_sparse_prefill_rows(Ps, cfg, m, 5, 5, ws)
    with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
        bf.bfla_sparse_prefill_rows(Ps, cfg, m, 0, B * Hkv * Tq + 1, ws)


def test_balanced_layer_single_rank_nccl():
    """The f2 strong-scaling layer (parallel.BalancedLayer: head-group masks on strided views, NCCL
    list all-gather, host slice bounds, sliced prefill into a zeroed O, O all-reduce) through a real
    one-rank NCCL group equals the unsharded whole path bit for bit."""
    import socket

    import torch.distributed as dist
    from paper_2605_12193_b200 import parallel

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        prob = workloads.structured(15, B=2, Hq=8, Hkv=2, Nq=2100, Nkv=2100, d=128, block=256)
        q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
        cfg = bf.Config(b=256, g=64, eta=8, rho=0.1, seed=4)
        o_ref, _ = bf.prefill(q, k, v, cfg)
        o = torch.full_like(q, 3.0)
        layer = parallel.BalancedLayer(q, k, v, o, cfg, 0, 1)
        layer.run()
        torch.cuda.synchronize()
        assert layer.bounds == (0, 2 * 2 * 33)
        assert torch.equal(o, o_ref)
        # the fused exchange (symmetric-memory O, mirrored slice stores + device barrier): no peers at world 1
        try:
            peer = parallel.PeerFullOutput(q.shape, 1, 0, q.device)
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"torch symmetric memory unavailable: {e}")
        peer.o.fill_(3.0)
        layer2 = parallel.BalancedLayer(q, k, v, peer.o, cfg, 0, 1, peer_out=peer)
        layer2.run()
        torch.cuda.synchronize()
        assert torch.equal(peer.o, o_ref)
    finally:
        dist.destroy_process_group()


def test_cuda_graph_capture_of_whole_path():
    """The library never synchronises or allocates, so one layer (Stage 1 with the side-stream norms and
    the recompute, Stage 2, sparse prefill with its dynamic-scheduling counter) captures into a CUDA
    graph; replays on new inputs written into the captured buffers give the eager results bit for bit."""
    prob = workloads.structured(16, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128, block=256)
    prob2 = workloads.structured(17, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128, block=256)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o = torch.empty_like(q)
    cfg = bf.Config(b=256, g=64, eta=8, rho=0.1, seed=3)
    P = bf.make_problem(q, k, v, o)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg)

    def layer():
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill(P, cfg, m, ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        layer()  # warm-up outside capture (function attributes, tensor maps)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    n0 = bf.kernel_launches()
    with torch.cuda.graph(graph):
        layer()
    assert bf.kernel_launches() - n0 >= 5
    outs = []
    for src in (prob, prob2):
        q.copy_(src.q.cuda()), k.copy_(src.k.cuda()), v.copy_(src.v.cuda())
        graph.replay()
        torch.cuda.synchronize()
        got = (o.clone(), m.tile_count.clone(), m.coarse_bits.clone())
        layer()
        torch.cuda.synchronize()
        assert torch.equal(got[0], o) and torch.equal(got[1], m.tile_count) and torch.equal(got[2], m.coarse_bits)
        outs.append(got[0])
    assert not torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("paged", [0, 16])
def test_chunked_prefill_tensor_core_stage1(paged):
    """Aligned chunked prefill (the vLLM case: N_c > 0 with n_q, n_kv multiples of g) takes the
    tensor-core Stage-1 path (tcgen05 scores + certification + canonical recompute); masks bit-exact
    against the oracle and equal to the all-canonical path, O on sampled rows within tolerance.
    n_q = 8192 queries attend to n_kv = 32768 keys (N_c = 24576, Eq. 11-13, R18)."""
    Hq, Hkv, Nq, Nkv, d = 8, 2, 8192, 32768, 128
    prob = workloads.structured(18, B=1, Hq=Hq, Hkv=Hkv, Nq=Nq, Nkv=Nkv, d=d, block=256)
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, rho=0.1, seed=11)
    n0 = bf.kernel_launches()
    fast = run_gpu(prob, cfg, paged_page=paged, lse=True)
    n_fast = bf.kernel_launches() - n0
    n0 = bf.kernel_launches()
    canon = run_gpu(prob, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), paged_page=paged, lse=False)
    n_canon = bf.kernel_launches() - n0
    # the AUTO call ran the tensor-core chain (norms + tcgen05 scores + select + recompute + re-select),
    # not the canonical SIMT fallback (scores + select)
    assert n_fast > n_canon, (n_fast, n_canon)
    assert np.array_equal(fast["coarse"], canon["coarse"]) and np.array_equal(fast["labels"], canon["labels"])
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(fast, ref, cfg)
    check_lists(fast, labels, Nq, Nkv, 64)
    tiles = list(range(0, Nq // 64, 16)) + [Nq // 64 - 1]
    rows = np.array([[p, i * 64 + r] for p in range(Hq) for i in tiles for r in range(64)], np.int32)
    (o_ref, lse_ref), = oracle_attention(prob, labels, 64, rows_per_req=[rows])
    og = fast["o"][0].float().cpu().numpy()[rows[:, 0], rows[:, 1]].astype(np.float64)
    err = np.abs(og - o_ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
    lg = fast["lse"][0].cpu().numpy()[rows[:, 0], rows[:, 1]]
    assert np.abs(lg - lse_ref).max() <= 1e-3
    print(f"chunked TC paged={paged}: kappa={fast['stats']['kept_tiles'] / fast['stats']['causal_tiles']:.3f} "
          f"flagged={fast['stats']['rows_flagged']} max-abs={err.max():.2e}")


@pytest.mark.parametrize("case", [
    dict(B=1, Hq=8, Hkv=2, Nq=5000, Nkv=5000, d=128),     # ragged N: 5000 mod 64 = 8, several score tiles
    dict(B=1, Hq=4, Hkv=2, Nq=3001, Nkv=9001, d=128),     # ragged chunk over a ragged context (N_c = 6000)
    dict(B=1, Hq=4, Hkv=2, Nq=4100, Nkv=4100, d=256),     # d = 256, partial group of 4 tokens
])
def test_ragged_tensor_core_stage1(case, b=256):
    """§8 f1 performance path: ragged N (n mod g != 0) takes the tensor-core Stage 1 (scores over full
    groups, canonical rewrite of the partial group's row and column), bit-exact against the oracle and
    against the all-canonical path, with more launches than the canonical chain (proof it ran)."""
    prob = workloads.structured(23, block=b, **case)
    cfg = bf.Config(b=b, g=64, gamma=0.95, eta=16, rho=0.1, seed=9)
    n0 = bf.kernel_launches()
    fast = run_gpu(prob, cfg, lse=False)
    n_fast = bf.kernel_launches() - n0
    n0 = bf.kernel_launches()
    canon = run_gpu(prob, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), lse=False)
    n_canon = bf.kernel_launches() - n0
    assert n_fast > n_canon, (n_fast, n_canon)
    assert np.array_equal(fast["coarse"], canon["coarse"]) and np.array_equal(fast["labels"], canon["labels"])
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(fast, ref, cfg)
    check_lists(fast, labels, case["Nq"], case["Nkv"], 64)


def test_varlen_tensor_core_stage1_large():
    """Varlen batch with ragged requests at sizes spanning many score tiles: tensor-core Stage 1 (full
    groups per request, padding garbage never read into a score) bit-exact against the oracle."""
    lens = [(4000, 6500), (2048, 2048), (1000, 5000)]
    prob, sl = _varlen_case(84, lens, Hq=8, Hkv=2)
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, rho=0.0, seed=2)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o = torch.zeros_like(q)
    P = bf.make_problem(q, k, v, o, seqlens=sl.cuda())
    m = bf.alloc_mask(P, cfg, labels=True)
    n0 = bf.kernel_launches()
    bf.bfla_block_mask(P, cfg, m, bf.alloc_workspace(P, cfg))
    n_fast = bf.kernel_launches() - n0
    bf.bfla_expand_rescue(P, cfg, m, None)
    mc = bf.alloc_mask(P, cfg)
    n0 = bf.kernel_launches()
    bf.bfla_block_mask(P, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), mc, bf.alloc_workspace(P, cfg))
    n_canon = bf.kernel_launches() - n0
    torch.cuda.synchronize()
    assert n_fast > n_canon
    assert torch.equal(mc.coarse_bits, m.coarse_bits)
    coarse, labels = m.coarse_dense().cpu().numpy(), m.tile_label.cpu().numpy()
    for r, (nq, nkv) in enumerate(lens):
        qf, kf = f32(prob.q[r])[:, :nq], f32(prob.k[r])[:, :nkv]
        ref = oracle.mask_pipeline(qf, kf, b=256, g=64, T=64, gamma=0.95, eta=16, rho=0.0, seed=2)
        Lq, Lkv = ref["coarse"].shape[1:]
        assert np.array_equal(coarse[r, :, :Lq, :Lkv], ref["coarse"]), r
        Tq, Tkv = ref["labels"].shape[1:]
        assert np.array_equal(labels[r, :, :Tq, :Tkv], ref["labels"]), r


@pytest.mark.parametrize("d", [128, 256])
def test_group_count_16_tensor_core(d):
    """§8 f3: G = b/g = 16 — the paper's b = 1024, g = 64 row of Tab.mask — on the tensor-core
    Stage 1 (the score epilogue max-pools 16 x 16 group pairs), bit-exact against the oracle and the
    canonical path (which takes the any-G SIMT kernel)."""
    prob = workloads.structured(31, B=1, Hq=4, Hkv=2, Nq=6144, Nkv=6144, d=d, block=1024)
    cfg = bf.Config(b=1024, g=64, gamma=0.99, eta=16, rho=0.1, seed=4)
    fast = run_gpu(prob, cfg, lse=False)
    canon = run_gpu(prob, dataclasses.replace(cfg, scores=bf.SCORES_CANONICAL), lse=False)
    assert np.array_equal(fast["coarse"], canon["coarse"]) and np.array_equal(fast["labels"], canon["labels"])
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(fast, ref, cfg)
    check_lists(fast, labels, 6144, 6144, 64)
    # G = 16 with g = 16 (b = 256): the recompute kernels' 16 chains per thread, forced through the band
    cfg2 = bf.Config(b=256, g=16, gamma=0.95, eta=0, certify_slack=3000.0)
    prob2 = workloads.gaussian(32, B=1, Hq=2, Hkv=1, Nq=2048, Nkv=2048, d=d, sigma=0.7)
    g2 = run_gpu(prob2, cfg2, lse=False)
    assert g2["stats"]["rows_flagged"] > 0
    _check_masks(g2, oracle_masks(prob2, cfg2), cfg2)


@pytest.mark.parametrize("b,n", [(64, 1000), (128, 1536)])
def test_group_size_one_exact_block_max(b, n):
    """§8 f3: g = 1 — Eq. 10 becomes the exact block max of Q K^T (G = b groups of one token) — on the
    any-G canonical kernel; bit-exact against the oracle, ragged tail included."""
    prob = workloads.gaussian(33, B=1, Hq=4, Hkv=2, Nq=n, Nkv=n, d=128, sigma=0.6)
    cfg = bf.Config(b=b, g=1, gamma=0.95, eta=4, rho=0.0, seed=1)
    gpu = run_gpu(prob, cfg)
    ref = oracle_masks(prob, cfg)
    labels = _check_masks(gpu, ref, cfg)
    (o_ref, _), = oracle_attention(prob, labels, 64)
    compare_o(gpu["o"][0], o_ref, f"g=1 b={b}")


@pytest.mark.parametrize("case", ["d128", "d256", "varlen", "rows", "paged"])
def test_mirrored_prefill_fused_exchange(case):
    """§8 f2 fused exchange: bfla_sparse_prefill_mirrored stores every O / LSE row into each mirror as
    well (on a multi-GPU box the mirrors are peers' symmetric-memory buffers; here, two local buffers).
    Mirrors and the local O must equal the plain sparse prefill bit for bit — TMA-store epilogue
    (d128, rows, paged), per-thread stores (d256, varlen) — and a row slice writes only its rows."""
    d = 256 if case == "d256" else 128
    if case == "varlen":
        prob, sl = _varlen_case(91, [(1500, 3000), (700, 700)], Hq=8, Hkv=2)
    else:
        prob, sl = workloads.structured(41, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=d, block=256), None
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, rho=0.1, seed=3)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    B, Hq, Nq, _ = q.shape
    o_ref = torch.zeros_like(q)
    l_ref = torch.zeros(B, Hq, Nq, dtype=torch.float32, device="cuda")
    if case == "paged":
        kc, vc, pt = workloads.paged(k, v, 16, seed=9, extra_pages=2)
        mk = lambda o, l: bf.make_problem(q, kc, vc, o, l, page_table=pt, n_kv=k.shape[2])
    else:
        mk = lambda o, l: bf.make_problem(q, k, v, o, l, seqlens=None if sl is None else sl.cuda())
    P = mk(o_ref, l_ref)
    ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    o = torch.zeros_like(q)
    l = torch.zeros_like(l_ref)
    mo = [torch.zeros_like(q) for _ in range(2)]
    ml = [torch.zeros_like(l_ref) for _ in range(2)]
    P2 = mk(o, l)
    rows = (0, 0)
    if case == "rows":
        Tq = -(-Nq // 64)
        rows = (Tq // 3, 2 * Tq)  # part of head group 0 and all of head group 1 (LPT order)
    n0 = bf.kernel_launches()
    bf.bfla_sparse_prefill_mirrored(P2, cfg, m, mo, ml, rows=rows, ws=ws)
    torch.cuda.synchronize()
    assert bf.kernel_launches() - n0 == 1  # one kernel: the exchange is fused into its epilogue
    if case != "rows":
        for t, ref in [(o, o_ref)] + [(x, o_ref) for x in mo]:
            assert torch.equal(t, ref)
        for t in [l] + ml:
            assert torch.equal(t, l_ref)
        return
    # the slice's rows: (h, i) for LPT rho in [r0, r1) -> query heads h*m .. h*m+m-1, tokens i*64 ..
    Tq, m_ = -(-Nq // 64), Hq // 2
    want = torch.zeros(B, Hq, Nq, dtype=torch.bool, device="cuda")
    for rho in range(*rows):
        h, i = rho // Tq, Tq - 1 - rho % Tq
        want[:, h * m_:(h + 1) * m_, i * 64:(i + 1) * 64] = True
    for t in [o] + mo:
        assert torch.equal(t[want], o_ref[want]) and not t[~want].any()
    for t in [l] + ml:
        assert torch.equal(t[want], l_ref[want]) and not t[~want].any()


def test_peer_head_output_symmetric_memory_single_rank():
    """The fused-exchange plumbing on one rank: parallel.PeerHeadOutput allocates the rank-major O in
    torch symmetric memory and rendezvouses (no peers, so no mirrors); the mirrored prefill into its
    local chunk plus the device barrier equals the plain prefill.  On a one-GPU box without symmetric
    memory support the test is skipped (bench falls back to the NCCL all-gather, reported in its line)."""
    import socket

    import torch.distributed as dist
    from paper_2605_12193_b200 import parallel

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        prob = workloads.structured(16, B=1, Hq=8, Hkv=2, Nq=3072, Nkv=3072, d=128, block=256)
        q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
        cfg = bf.Config(b=256, g=64, eta=8, rho=0.1, seed=4)
        o_ref, _ = bf.prefill(q, k, v, cfg)
        try:
            hout = parallel.PeerHeadOutput(1, 8, 3072, 128, 1, 0, q.device)
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"torch symmetric memory unavailable: {e}")
        assert hout.mirrors == []
        P = bf.make_problem(q, k, v, hout.local)
        ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg)
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill_mirrored(P, cfg, m, hout.mirrors, ws=ws)
        hout.finish()
        torch.cuda.synchronize()
        assert torch.equal(hout.full, o_ref)
        # NVLS: the same through the buffer's multicast address (multimem.st), when the node has one
        try:
            hmc = parallel.PeerHeadOutput(1, 8, 3072, 128, 1, 0, q.device, multicast=True)
        except Exception as e:  # noqa: BLE001
            print(f"NVLS multicast unavailable on this node: {e}")
            return
        hmc.local.zero_()
        scratch = torch.zeros_like(q)  # local O of the call; the multicast stores fill hmc's buffer
        Pm = bf.make_problem(q, k, v, scratch)
        bf.bfla_sparse_prefill_mirrored(Pm, cfg, m, [], ws=ws, multicast_o=hmc.multicast_o)
        hmc.finish()
        torch.cuda.synchronize()
        assert torch.equal(scratch, o_ref) and torch.equal(hmc.full, o_ref)
    finally:
        dist.destroy_process_group()


def test_ragged_tensor_core_stage1_large_blocks():
    """Ragged N at b = 1024 (G = 16: the partial-group fixup reads keys from global memory, the block does
    not fit the staged layout) and d = 256 at b = 512 (same), bit-exact as above."""
    test_ragged_tensor_core_stage1(dict(B=1, Hq=4, Hkv=2, Nq=5000, Nkv=5000, d=128), b=1024)
    test_ragged_tensor_core_stage1(dict(B=1, Hq=4, Hkv=2, Nq=3100, Nkv=3100, d=256), b=512)


@pytest.mark.parametrize("d,parts", [(128, 3), (256, 2), (128, 5)])
def test_split_kv_partials_merge(d, parts):
    """§8 f2 split-KV: the sparse prefill restricted to KV-tile ranges (bfla_sparse_prefill_kvrange) and
    the LSE merge (bfla_merge_partials) reproduce the unsplit O within bf16 rounding and LSE to 1e-5
    relative, and the oracle within the contract tolerance; rows with no kept tile in a range get
    LSE = -inf there and still merge exactly."""
    from paper_2605_12193_b200 import parallel

    prob = workloads.structured(44, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=d, block=256)
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, rho=0.1, seed=7)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o_ref = torch.empty_like(q)
    l_ref = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    P = bf.make_problem(q, k, v, o_ref, l_ref)
    ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg, labels=True)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    ranges = parallel.split_kv_ranges(m.Tkv, parts)
    o_parts, l_parts = [], []
    for a, b_ in ranges:
        o_k = torch.empty_like(q)
        l_k = torch.empty_like(l_ref)
        bf.bfla_sparse_prefill_kvrange(bf.make_problem(q, k, v, o_k, l_k), cfg, m, a, b_, ws=ws)
        o_parts.append(o_k)
        l_parts.append(l_k)
    torch.cuda.synchronize()
    assert any(bool((x == -float("inf")).any()) for x in l_parts)  # some rows have nothing in a range
    o = torch.empty_like(q)
    l = torch.empty_like(l_ref)
    bf.bfla_merge_partials(bf.make_problem(q, k, v, o, l), o_parts, l_parts)
    torch.cuda.synchronize()
    err = (o.float() - o_ref.float()).abs()
    assert err.max().item() <= 1.6e-2 and err.mean().item() <= 1e-3, (err.max().item(), err.mean().item())
    assert torch.allclose(l, l_ref, rtol=1e-5, atol=1e-5)
    labels = m.tile_label.cpu().numpy()
    rows = np.array([[p_, t] for p_ in range(8) for t in range(0, 4096, 37)], np.int32)
    (o_or, lse_or), = oracle_attention(prob, labels, 64, rows_per_req=[rows])
    og = o[0].float().cpu().numpy()[rows[:, 0], rows[:, 1]].astype(np.float64)
    e2 = np.abs(og - o_or)
    assert e2.max() <= 2e-2 and e2.mean() <= 2e-3, (e2.max(), e2.mean())


def test_split_kv_on_a_row_slice():
    """(row slice x KV range) pieces — what a scheduler hands out for rows too long for one rank: the
    pieces of one LPT row slice split into 3 KV ranges merge to the unsplit O on those rows and leave
    every other row untouched."""
    from paper_2605_12193_b200 import parallel

    prob = workloads.structured(45, B=1, Hq=8, Hkv=2, Nq=3072, Nkv=3072, d=128, block=256)
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, seed=8)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o_ref = torch.empty_like(q)
    l_ref = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    P = bf.make_problem(q, k, v, o_ref, l_ref)
    ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    Tq = m.Tq
    rows = (3, Tq + 5)  # tail of head group 0 (its longest rows) and the start of group 1
    o_parts, l_parts = [], []
    for a, b_ in parallel.split_kv_ranges(m.Tkv, 3):
        o_k = torch.zeros_like(q)
        l_k = torch.full_like(l_ref, -float("inf"))
        bf.bfla_sparse_prefill_kvrange(bf.make_problem(q, k, v, o_k, l_k), cfg, m, a, b_, rows=rows, ws=ws)
        o_parts.append(o_k)
        l_parts.append(l_k)
    o = torch.zeros_like(q)
    l = torch.full_like(l_ref, -float("inf"))
    bf.bfla_merge_partials(bf.make_problem(q, k, v, o, l), o_parts, l_parts)
    torch.cuda.synchronize()
    want = torch.zeros(q.shape[:3], dtype=torch.bool, device="cuda")
    for rho in range(*rows):
        h, i = rho // Tq, Tq - 1 - rho % Tq
        want[:, h * 4:(h + 1) * 4, i * 64:(i + 1) * 64] = True
    err = (o.float() - o_ref.float()).abs()[want]
    assert err.max().item() <= 1.6e-2 and err.mean().item() <= 1e-3
    assert torch.allclose(l[want], l_ref[want], rtol=1e-5, atol=1e-5)
    assert not o[~want].any() and bool((l[~want] == -float("inf")).all())


@pytest.mark.gpu
@pytest.mark.parametrize("parts,sms", [(8, 148), (4, 16), (2, 148)])
def test_split_kv_plan_executes_to_the_unsplit_output(parts, sms):
    """§8 f2 split-KV planner (parallel.plan_pieces): every rank's pieces — whole-row slices and
    (row slice x KV range) pieces of the rows longer than the per-SM share — run on one GPU into the
    plan's partial slots, and bfla_merge_partials gives the unsplit O within bf16 rounding and its LSE
    to 1e-5, and the oracle on sampled rows.  KV group 0 is diffuse (Q x 0.05: near-uniform block
    softmax), the case that splits."""
    from paper_2605_12193_b200 import parallel

    prob = workloads.structured(46, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128, block=256)
    prob.q[:, :4] *= 0.05
    cfg = bf.Config(b=256, g=64, gamma=0.95, eta=16, seed=9)
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o_ref = torch.empty_like(q)
    l_ref = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    P = bf.make_problem(q, k, v, o_ref, l_ref)
    ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg, labels=True)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    counts = m.tile_count.cpu().numpy()
    plan = parallel.plan_pieces(counts, parts, sms=sms)
    nslot = parallel.plan_slots(plan)
    if (parts, sms) == (8, 148):
        assert nslot > 1, "the diffuse head's long rows must be split"
    o_parts = [torch.zeros_like(q) for _ in range(nslot)]
    l_parts = [torch.full_like(l_ref, -float("inf")) for _ in range(nslot)]
    probs = [bf.make_problem(q, k, v, o_parts[s], l_parts[s]) for s in range(nslot)]
    for pieces in plan:
        parallel.run_plan(lambda s: probs[s], cfg, m, pieces, ws=ws)
    o = torch.empty_like(q)
    l = torch.empty_like(l_ref)
    bf.bfla_merge_partials(bf.make_problem(q, k, v, o, l), o_parts, l_parts)
    torch.cuda.synchronize()
    err = (o.float() - o_ref.float()).abs()
    assert err.max().item() <= 1.6e-2 and err.mean().item() <= 1e-3, (err.max().item(), err.mean().item())
    assert torch.allclose(l, l_ref, rtol=1e-5, atol=1e-5)
    if nslot == 1:
        assert torch.equal(o, o_ref)  # whole rows only: the merge of one part is exact
    labels = m.tile_label.cpu().numpy()
    rows = np.array([[p_, t] for p_ in (0, 3, 5) for t in range(0, 4096, 53)], np.int32)
    (o_or, _), = oracle_attention(prob, labels, 64, rows_per_req=[rows])
    og = o[0].float().cpu().numpy()[rows[:, 0], rows[:, 1]].astype(np.float64)
    e2 = np.abs(og - o_or)
    assert e2.max() <= 2e-2 and e2.mean() <= 2e-3, (e2.max(), e2.mean())
