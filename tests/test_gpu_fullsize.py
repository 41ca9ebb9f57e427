"""Full-size GPU parity at BASELINE.json's configurations, in the launch configuration bench.py times.

The whole-layer mask (coarse bits, tile labels, lists, counts) is compared bit for bit against the
oracle; O and LSE are compared on a deterministic sample of query tiles (every `stride`-th tile plus
the first and the last, all heads) — the oracle computes those rows one by one in fp64."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2605_12193_b200 as bf
import workloads
from gpu_util import ATOL_MAX, ATOL_MEAN, check_lists

pytestmark = pytest.mark.gpu

CASES = {
    # bench.py default: Llama-3.1-8B layer, 32K, strong operating point
    "llama8b-32k": dict(Hq=32, Hkv=8, d=128, N=32768, b=256, g=64, gamma=0.99, eta=16, rho=0.0, paged=0,
                        theta=5e5, seed=303),
    # Llama-3.1-8B layer at 128K (BASELINE.json configs[2], single-GPU slice of the sharded run)
    "llama8b-128k": dict(Hq=32, Hkv=8, d=128, N=131072, b=256, g=64, gamma=0.99, eta=16, rho=0.0, paged=0,
                         theta=5e5, seed=303),
    # Qwen3-32B-like, 64K, vLLM pages of 16, all rescues (BASELINE.json configs[3])
    "qwen32b-64k-paged": dict(Hq=64, Hkv=8, d=128, N=65536, b=256, g=64, gamma=0.99, eta=16, rho=0.1, paged=16,
                              theta=1e6, seed=404),
    # Gemma-like d=256 GQA shape (BASELINE.json configs[4]) at 32K and at the top of its 4K-128K sweep
    "gemma-d256-32k": dict(Hq=16, Hkv=8, d=256, N=32768, b=256, g=64, gamma=0.99, eta=16, rho=0.0, paged=0,
                           theta=1e6, seed=505),
    "gemma-d256-128k": dict(Hq=16, Hkv=8, d=256, N=131072, b=256, g=64, gamma=0.99, eta=16, rho=0.0, paged=0,
                            theta=1e6, seed=505),
    "gemma-d256-128k-ratio0.1": dict(Hq=16, Hkv=8, d=256, N=131072, b=256, g=64, gamma=0.99, eta=16, rho=0.0,
                                     paged=0, theta=1e6, seed=505, keep_ratio=0.1),
    # the Llama-32K keep-mass threshold sweep of BASELINE.json configs[1] (Tab.mask gamma values) and
    # the north_star's keep-ratio rule at the same shape
    "llama8b-32k-gamma0.9": dict(Hq=32, Hkv=8, d=128, N=32768, b=256, g=64, gamma=0.9, eta=16, rho=0.0, paged=0,
                                 theta=5e5, seed=303),
    "llama8b-32k-gamma0.95": dict(Hq=32, Hkv=8, d=128, N=32768, b=256, g=64, gamma=0.95, eta=16, rho=0.0, paged=0,
                                  theta=5e5, seed=303),
    "llama8b-32k-gamma0.999": dict(Hq=32, Hkv=8, d=128, N=32768, b=256, g=64, gamma=0.999, eta=16, rho=0.0,
                                   paged=0, theta=5e5, seed=303),
    "llama8b-32k-ratio0.1": dict(Hq=32, Hkv=8, d=128, N=32768, b=256, g=64, gamma=0.99, eta=16, rho=0.0, paged=0,
                                 theta=5e5, seed=303, keep_ratio=0.1),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize(name):
    c = CASES[name]
    ratio = c.get("keep_ratio", 0.0)
    sel = dict(select=bf.SELECT_RATIO, keep_ratio=ratio) if ratio else {}
    N, Hq, Hkv, d = c["N"], c["Hq"], c["Hkv"], c["d"]
    prob = workloads.structured(c["seed"], 1, Hq, Hkv, N, N, d, block=c["b"], theta=c["theta"], device="cuda")
    q, k, v = prob.q, prob.k, prob.v
    o = torch.empty_like(q)
    lse = torch.empty(1, Hq, N, dtype=torch.float32, device="cuda")
    cfg = bf.Config(b=c["b"], g=c["g"], T=64, gamma=c["gamma"], n_local=8, eta=c["eta"], rho=c["rho"], **sel)
    if c["paged"]:
        kc, vc, pt = workloads.paged(k, v, c["paged"], seed=c["seed"])
        P = bf.make_problem(q, kc, vc, o, lse, page_table=pt, n_kv=N)
    else:
        P = bf.make_problem(q, k, v, o, lse)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg, labels=True)
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    bf.bfla_sparse_prefill(P, cfg, m, ws)
    torch.cuda.synchronize()
    st = m.stats_dict()
    qf, kf, vf = (t[0].float().cpu().numpy() for t in (q, k, v))
    ref = oracle.mask_pipeline(qf, kf, b=c["b"], g=c["g"], T=64, gamma=c["gamma"], n_local=8, eta=c["eta"],
                               rho=c["rho"], select_mode=cfg.select, keep_ratio=cfg.keep_ratio)
    assert np.array_equal(m.coarse_dense()[0].cpu().numpy(), ref["coarse"]), "coarse mask mismatch"
    labels = m.tile_label[0].cpu().numpy()
    assert np.array_equal(labels, ref["labels"]), "tile mask mismatch"
    check_lists(dict(count=m.tile_count.cpu().numpy(), list=m.tile_list.cpu().numpy()), ref["labels"][None], N, N, 64)
    assert st["rows_exact_tie"] == int(ref["tie"].sum())
    kappa = st["kept_tiles"] / st["causal_tiles"]
    # O / LSE on sampled query tiles (all heads)
    Tq = N // 64
    stride = 64 if N <= 65536 else 256
    tiles = sorted(set(list(range(0, Tq, stride)) + [Tq - 1]))
    rows = np.array([[p, i * 64 + r] for p in range(Hq) for i in tiles for r in range(64)], np.int32)
    O_ref, lse_ref = oracle.masked_attention(qf, kf, vf, 1 / math.sqrt(d), ref["labels"], 64, rows)
    og = o[0].float().cpu().numpy()[rows[:, 0], rows[:, 1]].astype(np.float64)
    err = np.abs(og - O_ref)
    lg = lse[0].cpu().numpy()[rows[:, 0], rows[:, 1]]
    print(f"{name}: kappa={kappa:.4f} flagged={st['rows_flagged']} ties={st['rows_exact_tie']} "
          f"rows={len(rows)} max-abs={err.max():.3e} mean-abs={err.mean():.3e} lse-max={np.abs(lg - lse_ref).max():.2e}")
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN
    assert np.abs(lg - lse_ref).max() <= 1e-3
