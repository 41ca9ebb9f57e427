"""Multi-GPU partitioning of the BFLA hot path.

Every stage of the path is independent per (request r, KV head h): Stage 1 ORs only within the head
group H_h (Eq. 8, Eq. 20), Stage 2 and the sparse prefill (Eq. 27) are per (r, h).  So a layer shards
by KV-head groups (and by request) with no cross-GPU reduction; the only exchange is an all-gather
of O when every rank needs the full output.  Random rescue psi (Eq. 25) takes the GLOBAL KV head
index, passed as `head_offset`, so a sharded mask equals the unsharded one bit for bit.

Host-side plumbing only (views, offsets, the collective); all compute runs in libbfla.so.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(h_kv: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous KV-head slice [h0, h1) of `rank`; the query heads are [h0*m, h1*m)."""
    if h_kv % world:
        raise ValueError(f"h_kv={h_kv} is not divisible by world={world}")
    per = h_kv // world
    return rank * per, (rank + 1) * per


def shard_views(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, rank: int, world: int):
    """Zero-copy head-first views of this rank's shard: (q, k, v, head_offset).

    q: [B, Hq, Nq, d], k/v: [B, Hkv, Nkv, d] (head-first, so a head slice is a strided view)."""
    h_kv = k.shape[1]
    m = q.shape[1] // h_kv
    h0, h1 = head_range(h_kv, world, rank)
    return q[:, h0 * m:h1 * m], k[:, h0:h1], v[:, h0:h1], h0


def gather_heads(o_shard: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather head-sharded outputs [B, Hq/world, N, d] into [B, Hq, N, d] (rank order = head order).

    NCCL: one all_gather_into_tensor into a [world, B, Hq/world, N, d] buffer; other backends
    (gloo, used by the CPU tests) fall back to the list form of all_gather."""
    o_shard = o_shard.contiguous()
    B, hs, N, d = o_shard.shape
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world,) + tuple(o_shard.shape), dtype=o_shard.dtype, device=o_shard.device)
        dist.all_gather_into_tensor(buf, o_shard, group=group)
        parts = buf.unbind(0)
    else:
        parts = [torch.empty_like(o_shard) for _ in range(world)]
        dist.all_gather(parts, o_shard, group=group)
    return torch.cat(parts, dim=1)


def request_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Request (batch) slice for request-level sharding: requests are fully independent."""
    per = -(-batch // world)
    return min(batch, rank * per), min(batch, (rank + 1) * per)
