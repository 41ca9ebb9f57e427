"""Seeded synthetic inputs for BFLA — shared by the oracle tests, the GPU parity tests and bench.

This module holds NONE of the method's arithmetic (no pooling, scoring, softmax, selection,
rescue or attention): it only draws Q/K/V tensors and builds paged-KV layouts.  Both sides
(oracle/ and the CUDA path) consume what it returns; neither is imported here.

Recipes:
  gaussian(sigma)  i.i.d. N(0, sigma^2) Q/K/V — parity stress (sigma=1 winner-take-all,
                   sigma<1 keeps many blocks per row and exercises sort/prefix/ties).
  structured       model-like attention: per-KV-head shared content vector + RoPE (locality,
                   decays with |t - s|), attention sinks on the first tokens, and scattered
                   heavy KV blocks that a random subset of later query blocks attends to.
                   This is the paper's workload shape (sinks + local + scattered heavy blocks,
                   BASELINE.json north_star); the paper's own inputs (LongBench through real
                   models) are out of scope.
Paged K/V follows vLLM's cache layout [num_pages, page_size, H_kv, d] with a seeded
Fisher-Yates page permutation as the page table.
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass
class Problem:
    q: torch.Tensor  # [B, Hq, Nq, d] bf16
    k: torch.Tensor  # [B, Hkv, Nkv, d] bf16
    v: torch.Tensor  # [B, Hkv, Nkv, d] bf16

    @property
    def shape(self):
        B, Hq, Nq, d = self.q.shape
        return B, Hq, self.k.shape[1], Nq, self.k.shape[2], d


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def gaussian(seed: int, B: int, Hq: int, Hkv: int, Nq: int, Nkv: int, d: int, sigma: float = 1.0,
             device="cpu") -> Problem:
    g = _gen(device, seed)
    mk = lambda H, N: (torch.randn(B, H, N, d, generator=g, device=device) * sigma).to(torch.bfloat16)
    return Problem(mk(Hq, Nq), mk(Hkv, Nkv), mk(Hkv, Nkv))


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    d = x.shape[-1]
    half = d // 2
    inv = theta ** (-torch.arange(half, device=x.device, dtype=torch.float32) / half)
    ang = pos.to(torch.float32)[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], dim=-1)


def structured(seed: int, B: int, Hq: int, Hkv: int, Nq: int, Nkv: int, d: int, *,
               block: int = 256, theta: float = 5e5, a_loc: float = 0.6, beta_sink: float = 1.0,
               beta_heavy: float = 0.6, n_heavy: int = 8, p_act: float = 0.25, n_sink_tok: int = 4,
               device="cpu") -> Problem:
    """Model-like Q/K/V (sinks + locality + scattered heavy blocks), bf16, post-RoPE."""
    g = _gen(device, seed)
    m = Hq // Hkv
    n_c = Nkv - Nq
    f32 = torch.float32
    q = torch.randn(B, Hq, Nq, d, generator=g, device=device)
    k = torch.randn(B, Hkv, Nkv, d, generator=g, device=device)
    v = torch.randn(B, Hkv, Nkv, d, generator=g, device=device)
    # locality: a shared per-KV-head content vector in q (whole group) and k; RoPE turns the
    # common component into a term that peaks at t == s and decays with the distance.
    c = torch.randn(B, Hkv, 1, d, generator=g, device=device)
    k = k + a_loc * c
    q = q + a_loc * c.repeat_interleave(m, dim=1)
    q = _rope(q, torch.arange(n_c, n_c + Nq, device=device), theta)
    k = _rope(k, torch.arange(Nkv, device=device), theta)
    # sinks: the first tokens' keys align with the group's mean query direction
    qm = q.view(B, Hkv, m, Nq, d).mean(dim=(2, 3))  # [B, Hkv, d]
    w = qm / qm.norm(dim=-1, keepdim=True).clamp_min(1e-6)
    ns = min(n_sink_tok, Nkv)
    k[:, :, :ns] += beta_sink * math.sqrt(d) * w[:, :, None, :]
    # scattered heavy blocks: per KV head, n_heavy block-aligned KV blocks carry a direction
    # w_r; each query head of the group attends it from a random subset of later query blocks.
    L_kv = max(1, Nkv // block)
    L_q = max(1, -(-Nq // block))
    for bb in range(B):
        for h in range(Hkv):
            blocks = torch.randint(0, L_kv, (n_heavy,), generator=g, device=device).tolist()
            dirs = torch.randn(n_heavy, d, generator=g, device=device)
            dirs = dirs / dirs.norm(dim=-1, keepdim=True)
            for r, jb in enumerate(blocks):
                s0, s1 = jb * block, min(Nkv, (jb + 1) * block)
                k[bb, h, s0:s1] += beta_heavy * math.sqrt(d) * dirs[r]
                for p in range(h * m, (h + 1) * m):
                    act = torch.rand(L_q, generator=g, device=device) < p_act
                    for i in torch.nonzero(act).flatten().tolist():
                        t0, t1 = i * block, min(Nq, (i + 1) * block)
                        if n_c + t0 < s0:  # only later query blocks (causal)
                            continue
                        q[bb, p, t0:t1] += beta_heavy * math.sqrt(d) * dirs[r]
    bf = torch.bfloat16
    return Problem(q.to(f32).to(bf), k.to(f32).to(bf), v.to(f32).to(bf))


def paged(k: torch.Tensor, v: torch.Tensor, page_size: int, seed: int, extra_pages: int = 0):
    """vLLM-style paged cache: returns (k_cache, v_cache [P, page, Hkv, d], page_table [B, maxp] int32).

    Logical page n of request b lives at physical page page_table[b, n]; physical pages are a
    seeded Fisher-Yates permutation of all pages (plus `extra_pages` unused ones).
    """
    B, Hkv, N, d = k.shape
    maxp = -(-N // page_size)
    npages = B * maxp + extra_pages
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    perm = torch.randperm(npages, generator=g)
    table = perm[: B * maxp].view(B, maxp).to(torch.int32)
    kc = torch.zeros(npages, page_size, Hkv, d, dtype=k.dtype, device=k.device)
    vc = torch.zeros_like(kc)
    pad = maxp * page_size - N
    kp = torch.nn.functional.pad(k, (0, 0, 0, pad)).view(B, Hkv, maxp, page_size, d).permute(0, 2, 3, 1, 4)
    vp = torch.nn.functional.pad(v, (0, 0, 0, pad)).view(B, Hkv, maxp, page_size, d).permute(0, 2, 3, 1, 4)
    idx = table.view(-1).long().to(k.device)
    kc[idx] = kp.reshape(B * maxp, page_size, Hkv, d)
    vc[idx] = vp.reshape(B * maxp, page_size, Hkv, d)
    return kc, vc, table.to(k.device)
