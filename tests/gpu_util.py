"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI and the oracle on
the same seeded inputs, and compare.  Test infrastructure (may import oracle/)."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
import paper_2605_12193_b200 as bf
import workloads

ATOL_MAX, ATOL_MEAN = 2e-2, 2e-3  # BASELINE.json: bf16 in, fp32 accumulation


def f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def run_gpu(prob: workloads.Problem, cfg, *, paged_page: int = 0, seed: int = 0, lse: bool = True,
            labels: bool = True, kept_mass: bool = False, head_offset: int = 0):
    """Stage 1 -> Stage 2 -> sparse prefill through the four ABI calls; returns tensors on CPU."""
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    B, Hq, Nq, d = q.shape
    Nkv = k.shape[2]
    o = torch.empty_like(q)
    l = torch.empty(B, Hq, Nq, dtype=torch.float32, device="cuda") if lse else None
    if paged_page:
        kc, vc, pt = workloads.paged(k, v, paged_page, seed=seed + 7, extra_pages=3)
        P = bf.make_problem(q, kc, vc, o, l, page_table=pt, n_kv=Nkv, head_offset=head_offset)
    else:
        P = bf.make_problem(q, k, v, o, l, head_offset=head_offset)
    out = {}
    if cfg is None:
        bf.bfla_prefill(P, None, None, None)
    else:
        ws = bf.alloc_workspace(P, cfg)
        m = bf.alloc_mask(P, cfg, labels=labels, kept_mass=kept_mass)
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill(P, cfg, m, ws)
        torch.cuda.synchronize()
        out["ws"] = ws
        out["mask"] = m
        out["coarse"] = m.coarse_dense().cpu().numpy()
        out["tiles"] = m.tile_dense().cpu().numpy()
        out["labels"] = m.tile_label.cpu().numpy() if labels else None
        out["count"] = m.tile_count.cpu().numpy()
        out["list"] = m.tile_list.cpu().numpy()
        out["kept_mass"] = m.kept_mass.cpu().numpy() if kept_mass else None
        out["stats"] = m.stats_dict()
    torch.cuda.synchronize()
    out["o"] = o
    out["lse"] = l
    return out


def oracle_masks(prob: workloads.Problem, cfg, head_offset: int = 0):
    """Per request r: the oracle's mask pipeline (Stage 1 + Stage 2)."""
    res = []
    for r in range(prob.q.shape[0]):
        res.append(oracle.mask_pipeline(f32(prob.q[r]), f32(prob.k[r]), b=cfg.b, g=cfg.g, T=cfg.T, pool=cfg.pool,
                                        gamma=cfg.gamma, select_mode=cfg.select, keep_ratio=cfg.keep_ratio,
                                        n_sink=cfg.n_sink, n_local=cfg.n_local, eta=cfg.eta, rho=cfg.rho,
                                        seed=cfg.seed, head_offset=head_offset))
    return res


def causal_row_counts(Nq: int, Nkv: int, T: int) -> np.ndarray:
    Tq, Tkv = -(-Nq // T), -(-Nkv // T)
    return np.array([sum(oracle.causal(i, j, T, Nq, Nkv) for j in range(Tkv)) for i in range(Tq)])


def check_lists(gpu: dict, labels_all: np.ndarray, Nq: int, Nkv: int, T: int):
    """labels_all [B, Hkv, Tq, Tkv] from the oracle -> expected counts and per-row lists at the
    documented causal offsets (computed here independently by a running sum)."""
    B, Hkv, Tq, _ = labels_all.shape
    rc = causal_row_counts(Nq, Nkv, T)
    offs = np.concatenate([[0], np.cumsum(rc)])
    per_head = offs[-1]
    for r in range(B):
        for h in range(Hkv):
            for i in range(Tq):
                want = np.nonzero(labels_all[r, h, i])[0]
                assert gpu["count"][r, h, i] == len(want), (r, h, i)
                base = (r * Hkv + h) * per_head + offs[i]
                assert np.array_equal(gpu["list"][base:base + len(want)], want), (r, h, i)


def oracle_attention(prob: workloads.Problem, labels_all, T: int, rows_per_req=None, scale=None):
    """fp64 oracle O (and LSE) for request r; labels_all None -> dense causal."""
    B, Hq, Nq, d = prob.q.shape
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    outs = []
    for r in range(B):
        lab = None if labels_all is None else labels_all[r]
        rows = None if rows_per_req is None else rows_per_req[r]
        outs.append(oracle.masked_attention(f32(prob.q[r]), f32(prob.k[r]), f32(prob.v[r]), scale, lab, T, rows))
    return outs


def compare_o(o_gpu: torch.Tensor, o_ref: np.ndarray, what: str = ""):
    og = o_gpu.float().cpu().numpy().astype(np.float64)
    err = np.abs(og - o_ref)
    mx, mean = float(err.max()), float(err.mean())
    assert mx <= ATOL_MAX and mean <= ATOL_MEAN, f"{what}: max-abs {mx:.3e} mean-abs {mean:.3e} max|O| {np.abs(o_ref).max():.2f}"
    return mx, mean
