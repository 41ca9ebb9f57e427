"""paper_2605_12193_b200 — B200-native (sm_100a) hot path of BFLA (arXiv 2605.12193).

Python binding of the C ABI in include/bfla.h (libbfla.so).  PyTorch supplies device memory and
streams only; every step of the path (Stage 1, Stage 2, sparse prefill) runs in the library's
CUDA kernels.  Names follow the ABI: bfla_block_mask, bfla_expand_rescue, bfla_sparse_prefill,
bfla_prefill, bfla_workspace_size, bfla_tile_list_capacity.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Optional

import torch

from . import _lib
from ._lib import (KV_CONTIGUOUS, KV_PAGED, MASK_PER_KV_HEAD, MASK_PER_Q_HEAD, POOL_FLATTEN, POOL_MEAN, SCORES_AUTO,
                   SCORES_CANONICAL, SELECT_MASS, SELECT_RATIO, bfla_config,
                   bfla_mask, bfla_problem, bfla_stats, check, lib)

__all__ = ["bfla_sparse_prefill_mirrored", "bfla_sparse_prefill_kvrange", "bfla_merge_partials", "Config", "Problem", "Mask", "make_problem", "alloc_mask", "alloc_workspace", "bfla_workspace_size",
           "bfla_tile_list_capacity", "bfla_block_mask", "bfla_expand_rescue", "bfla_sparse_prefill",
           "bfla_sparse_prefill_rows", "bfla_balance_rows", "bfla_prefill", "prefill", "kernel_launches", "POOL_FLATTEN", "POOL_MEAN", "SELECT_MASS", "SELECT_RATIO", "SCORES_AUTO",
           "SCORES_CANONICAL", "MASK_PER_KV_HEAD", "MASK_PER_Q_HEAD"]


@dataclasses.dataclass
class Config:
    """Method knobs (bfla_config).  Defaults: the paper's strong operating point."""
    b: int = 256
    g: int = 64
    T: int = 64
    pool: int = POOL_FLATTEN
    select: int = SELECT_MASS
    gamma: float = 0.99
    keep_ratio: float = 1.0
    n_sink: int = 1
    n_local: int = 8
    eta: int = 16
    rho: float = 0.0
    seed: int = 0
    scores: int = SCORES_AUTO
    mask_groups: int = MASK_PER_KV_HEAD  # MASK_PER_Q_HEAD: Eq. 18 literal, one mask per query head
    certify_slack: float = 0.0  # >= 1 widens the certification bound (tests: forces the recompute)

    def c(self) -> bfla_config:
        return bfla_config(self.b, self.g, self.T, self.pool, self.select, self.gamma, self.keep_ratio,
                           self.n_sink, self.n_local, self.eta, self.rho, self.seed, self.scores, self.mask_groups,
                           self.certify_slack)


@dataclasses.dataclass
class Problem:
    """bfla_problem plus the tensors it points into (kept alive here)."""
    c: bfla_problem
    tensors: tuple

    @property
    def shape(self):
        p = self.c
        return p.batch, p.h_q, p.h_kv, p.n_q, p.n_kv, p.head_dim


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def make_problem(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor,
                 lse: Optional[torch.Tensor] = None, *, softmax_scale: float = 0.0, head_offset: int = 0,
                 page_table: Optional[torch.Tensor] = None, n_kv: Optional[int] = None,
                 seqlens: Optional[torch.Tensor] = None) -> Problem:
    """q, o: [B, Hq, Nq, d] bf16 (strided views allowed, d contiguous).
    Contiguous K/V: k, v [B, Hkv, Nkv, d].  Paged (vLLM): k, v [num_pages, page_size, Hkv, d] and
    page_table int32 [B, max_pages]; n_kv must then be given.  seqlens (optional, int32 [B, 2] on the
    device): per-request (n_q_r, n_kv_r) of a variable-length batch padded to the tensor extents."""
    B, Hq, Nq, d = q.shape
    for t in (q, k, v, o):
        if t.dtype != torch.bfloat16 or not t.is_cuda or t.stride(-1) != 1:
            raise ValueError("q/k/v/o must be CUDA bf16 tensors with a contiguous last dim")
    p = bfla_problem()
    p.batch, p.h_q, p.head_dim, p.n_q = B, Hq, d, Nq
    p.softmax_scale = float(softmax_scale)
    p.head_offset = int(head_offset)
    p.q, p.o = _ptr(q), _ptr(o)
    p.q_stride[:] = list(q.stride()[:3])
    p.o_stride[:] = list(o.stride()[:3])
    p.lse = _ptr(lse)
    p.k, p.v = _ptr(k), _ptr(v)
    keep = [q, k, v, o]
    if lse is not None:
        keep.append(lse)
    if page_table is None:
        p.kv_layout = KV_CONTIGUOUS
        p.h_kv, p.n_kv = k.shape[1], k.shape[2]
        if k.stride() != v.stride():
            raise ValueError("k and v must share strides")
        p.kv_stride[:] = list(k.stride()[:3])
    else:
        if n_kv is None:
            raise ValueError("paged K/V needs n_kv")
        p.kv_layout = KV_PAGED
        num_pages, page_size, Hkv, _ = k.shape
        if not (k.is_contiguous() and v.is_contiguous()):
            raise ValueError("paged caches must be dense [num_pages, page_size, Hkv, d]")
        p.h_kv, p.n_kv = Hkv, int(n_kv)
        p.page_size, p.num_pages, p.max_pages_per_seq = page_size, num_pages, page_table.shape[1]
        pt = page_table.to(torch.int32).contiguous()
        p.page_table = _ptr(pt)
        keep.append(pt)
    if seqlens is not None:
        sl = seqlens.to(device=q.device, dtype=torch.int32).contiguous()
        if sl.shape != (B, 2):
            raise ValueError("seqlens must be [batch, 2] = (n_q_r, n_kv_r)")
        p.seqlens = _ptr(sl)
        keep.append(sl)
    return Problem(p, tuple(keep))


def bfla_workspace_size(problem: Problem, cfg: Optional[Config]) -> int:
    cc = None if cfg is None else ctypes.byref(cfg.c())
    return int(lib().bfla_workspace_size(ctypes.byref(problem.c), cc))


def bfla_tile_list_capacity(problem: Problem, cfg: Config) -> int:
    return int(lib().bfla_tile_list_capacity(ctypes.byref(problem.c), ctypes.byref(cfg.c())))


def alloc_workspace(problem: Problem, cfg: Optional[Config]) -> torch.Tensor:
    n = max(1, bfla_workspace_size(problem, cfg))
    return torch.empty(n, dtype=torch.uint8, device="cuda")


class Mask:
    """Caller-owned mask buffers (bfla_mask) as torch tensors."""

    def __init__(self, problem: Problem, cfg: Config, labels: bool = False, kept_mass: bool = False,
                 stats: bool = True):
        B, Hq, Hkv, Nq, Nkv, _ = problem.shape
        if cfg.mask_groups == MASK_PER_Q_HEAD:
            Hkv = Hq  # one mask group per query head
        dev = "cuda"
        cd = lambda a, b: -(-a // b)
        Lq, Lkv, Tq, Tkv = cd(Nq, cfg.b), cd(Nkv, cfg.b), cd(Nq, cfg.T), cd(Nkv, cfg.T)
        self.Lq, self.Lkv, self.Tq, self.Tkv = Lq, Lkv, Tq, Tkv
        cap = bfla_tile_list_capacity(problem, cfg)
        if cap < 0:  # the negated bfla_status of the invalid (problem, config)
            check(-cap, "bfla_tile_list_capacity")
        self.coarse_bits = torch.zeros(B, Hkv, Lq, cd(Lkv, 32), dtype=torch.int32, device=dev)
        self.tile_bits = torch.zeros(B, Hkv, Tq, cd(Tkv, 32), dtype=torch.int32, device=dev)
        self.tile_list = torch.zeros(max(1, cap), dtype=torch.int32, device=dev)
        self.tile_count = torch.zeros(B, Hkv, Tq, dtype=torch.int32, device=dev)
        self.tile_label = torch.zeros(B, Hkv, Tq, Tkv, dtype=torch.uint8, device=dev) if labels else None
        self.kept_mass = torch.zeros(B, Hq, Lq, dtype=torch.float32, device=dev) if kept_mass else None
        self.stats = torch.zeros(ctypes.sizeof(bfla_stats) // 8, dtype=torch.int64, device=dev) if stats else None
        self.cap = cap

    def c(self) -> bfla_mask:
        m = bfla_mask()
        m.coarse_bits, m.tile_bits = _ptr(self.coarse_bits), _ptr(self.tile_bits)
        m.tile_list, m.tile_list_capacity = _ptr(self.tile_list), self.cap
        m.tile_count = _ptr(self.tile_count)
        m.tile_label, m.kept_mass, m.stats = _ptr(self.tile_label), _ptr(self.kept_mass), _ptr(self.stats)
        return m

    def stats_dict(self) -> dict:
        s = self.stats.cpu().tolist()
        return dict(causal_tiles=s[0], kept_tiles=s[1], label=s[2:8], rows=s[8], rows_exact_tie=s[9],
                    blocks_kept=s[10], rows_flagged=s[11], rows_recomputed=s[12])

    def coarse_dense(self) -> torch.Tensor:
        """Unpack coarse_bits to a [B, Hkv, Lq, Lkv] uint8 tensor (test helper)."""
        return _unpack(self.coarse_bits, self.Lkv)

    def tile_dense(self) -> torch.Tensor:
        return _unpack(self.tile_bits, self.Tkv)


def _unpack(words: torch.Tensor, n: int) -> torch.Tensor:
    w = words.to(torch.int64) & 0xFFFFFFFF
    bits = (w.unsqueeze(-1) >> torch.arange(32, device=w.device)) & 1
    return bits.flatten(-2)[..., :n].to(torch.uint8)


def alloc_mask(problem: Problem, cfg: Config, **kw) -> Mask:
    return Mask(problem, cfg, **kw)


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def bfla_block_mask(problem: Problem, cfg: Config, mask: Mask, ws: torch.Tensor, stream=None) -> None:
    m = mask.c()
    check(lib().bfla_block_mask(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m), _ptr(ws),
                                ws.numel(), _stream(stream)), "bfla_block_mask")


def bfla_expand_rescue(problem: Problem, cfg: Config, mask: Mask, ws: Optional[torch.Tensor] = None,
                       stream=None) -> None:
    m = mask.c()
    check(lib().bfla_expand_rescue(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m), _ptr(ws),
                                   0 if ws is None else ws.numel(), _stream(stream)), "bfla_expand_rescue")


def bfla_sparse_prefill(problem: Problem, cfg: Config, mask: Mask, ws: Optional[torch.Tensor] = None,
                        stream=None) -> None:
    m = mask.c()
    check(lib().bfla_sparse_prefill(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m), _ptr(ws),
                                    0 if ws is None else ws.numel(), _stream(stream)), "bfla_sparse_prefill")


def bfla_sparse_prefill_rows(problem: Problem, cfg: Config, mask: Mask, row_begin: int, row_end: int,
                             ws: Optional[torch.Tensor] = None, stream=None) -> None:
    """Sparse prefill of the LPT-order rows [row_begin, row_end) only (include/bfla.h, §8 f2)."""
    m = mask.c()
    check(lib().bfla_sparse_prefill_rows(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m),
                                         int(row_begin), int(row_end), _ptr(ws), 0 if ws is None else ws.numel(),
                                         _stream(stream)), "bfla_sparse_prefill_rows")


def bfla_sparse_prefill_mirrored(problem: Problem, cfg: Config, mask: Mask, mirrors, lse_mirrors=None,
                                 rows: tuple[int, int] = (0, 0), ws: Optional[torch.Tensor] = None,
                                 stream=None, multicast_o: int = 0, multicast_lse: int = 0) -> None:
    """Sparse prefill whose epilogue also stores every O (+ LSE) row into each of `mirrors` (§8 f2 fused
    exchange, include/bfla.h).  mirrors: device tensors shaped like O, or raw device addresses (ints,
    e.g. peer-mapped symmetric-memory pointers) with O's layout; lse_mirrors likewise (or None).
    multicast_o / multicast_lse: NVLS multicast addresses (ints) written through multimem.st.
    rows = (0, 0): every row, else an LPT row slice as in bfla_sparse_prefill_rows."""
    mirrors = list(mirrors)
    if len(mirrors) > _lib.MAX_MIRRORS:
        raise ValueError(f"at most {_lib.MAX_MIRRORS} mirrors")
    mc = _lib.bfla_mirrors()
    mc.n = len(mirrors)
    keep = []
    for k, t in enumerate(mirrors):
        if isinstance(t, torch.Tensor):
            o = problem.tensors[3]
            if t.shape != o.shape or t.stride() != o.stride() or t.dtype != o.dtype or t.device != o.device:
                raise ValueError("an O mirror must have O's shape, strides and dtype")
            keep.append(t)
            mc.o[k] = t.data_ptr()
        else:
            mc.o[k] = int(t)
        if lse_mirrors is not None and lse_mirrors[k] is not None:
            lt = lse_mirrors[k]
            mc.lse[k] = lt.data_ptr() if isinstance(lt, torch.Tensor) else int(lt)
    mc.multicast_o = int(multicast_o) or None
    mc.multicast_lse = int(multicast_lse) or None
    m = mask.c()
    check(lib().bfla_sparse_prefill_mirrored(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m),
                                             int(rows[0]), int(rows[1]), ctypes.byref(mc), _ptr(ws),
                                             0 if ws is None else ws.numel(), _stream(stream)),
          "bfla_sparse_prefill_mirrored")


def bfla_sparse_prefill_kvrange(problem: Problem, cfg: Config, mask: Mask, kv_begin: int, kv_end: int,
                                rows: tuple[int, int] = (0, 0), ws: Optional[torch.Tensor] = None,
                                stream=None) -> None:
    """Split-KV partial: the sparse prefill over the kept tiles j in [kv_begin, kv_end) (mask tiles) only,
    for the LPT rows `rows` ((0, 0) = all); writes the range's normalised O and its LSE (problem must
    carry an LSE buffer)."""
    m = mask.c()
    check(lib().bfla_sparse_prefill_kvrange(ctypes.byref(problem.c), ctypes.byref(cfg.c()), ctypes.byref(m),
                                            int(kv_begin), int(kv_end), int(rows[0]), int(rows[1]), _ptr(ws),
                                            0 if ws is None else ws.numel(), _stream(stream)),
          "bfla_sparse_prefill_kvrange")


def bfla_merge_partials(problem: Problem, o_parts, lse_parts, stream=None) -> None:
    """O / LSE of problem from KV-range partials (tensors with O's / LSE's layout)."""
    if len(o_parts) != len(lse_parts) or not 1 <= len(o_parts) <= _lib.MAX_PARTS:
        raise ValueError(f"1..{_lib.MAX_PARTS} (O, LSE) partial pairs")
    pc = _lib.bfla_partials()
    pc.n = len(o_parts)
    for k, (o, l) in enumerate(zip(o_parts, lse_parts)):
        pc.o[k], pc.lse[k] = o.data_ptr(), l.data_ptr()
    check(lib().bfla_merge_partials(ctypes.byref(problem.c), ctypes.byref(pc), _stream(stream)),
          "bfla_merge_partials")


def bfla_balance_rows(tile_count, parts: int, row_overhead: int = 3) -> list[int]:
    """Cost-balanced slice bounds (parts + 1 of them) of the LPT row order; tile_count is a host
    [batch, h_kv, tq] int32 tensor/array (a copy of mask.tile_count).  Host-only library call."""
    t = torch.as_tensor(tile_count).to(torch.int32).contiguous().cpu()
    if t.dim() != 3:
        raise ValueError("tile_count must be [batch, h_kv, tq]")
    bounds = (ctypes.c_int64 * (parts + 1))()
    check(lib().bfla_balance_rows(ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_int32)), t.shape[0], t.shape[1],
                                  t.shape[2], int(row_overhead), int(parts), bounds), "bfla_balance_rows")
    return list(bounds)


def bfla_prefill(problem: Problem, cfg: Optional[Config], mask: Optional[Mask], ws: Optional[torch.Tensor],
                 stream=None) -> None:
    """Whole path (Stage 1 -> Stage 2 -> sparse prefill); cfg=None runs dense causal attention."""
    cc = None if cfg is None else ctypes.byref(cfg.c())
    mc = None
    if mask is not None:
        m = mask.c()
        mc = ctypes.byref(m)
    check(lib().bfla_prefill(ctypes.byref(problem.c), cc, mc, _ptr(ws), 0 if ws is None else ws.numel(),
                             _stream(stream)), "bfla_prefill")


def prefill(q, k, v, cfg: Optional[Config] = None, *, lse: bool = False, page_table=None, n_kv=None,
            softmax_scale: float = 0.0):
    """Convenience: allocate O (+LSE) and run bfla_prefill.  Returns (O, LSE or None)."""
    o = torch.empty_like(q)
    l = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device) if lse else None
    prob = make_problem(q, k, v, o, l, page_table=page_table, n_kv=n_kv, softmax_scale=softmax_scale)
    ws = alloc_workspace(prob, cfg) if cfg is not None else None
    bfla_prefill(prob, cfg, None, ws)
    return o, l


def kernel_launches() -> int:
    return int(lib().bfla_kernel_launches())
