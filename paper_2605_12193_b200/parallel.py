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


class HeadShardedOutput:
    """The layer's O in rank-major storage [world][B][Hq/world][N][d].

    Rank r's query heads [r*Hq/world, (r+1)*Hq/world) are ONE contiguous chunk (`local`, [B, Hq/world,
    N, d]), so the prefill kernel writes its shard straight into the full buffer and a single in-place
    all_gather_into_tensor assembles the layer: no staging buffer, no torch.cat, no copy.  `full` is
    the [B, Hq, N, d] view of the same storage (plain for B = 1; for B > 1 heads of different ranks are
    a further world-stride apart, so `full` is the 5-D [B, world, Hq/world, N, d] view)."""

    def __init__(self, B: int, Hq: int, N: int, d: int, world: int, rank: int, device, dtype=None):
        if Hq % world:
            raise ValueError(f"h_q={Hq} is not divisible by world={world}")
        self.world, self.rank = world, rank
        self.store = torch.empty(world, B, Hq // world, N, d, dtype=dtype or torch.bfloat16, device=device)
        self.local = self.store[rank]
        perm = self.store.permute(1, 0, 2, 3, 4)
        self.full = perm.reshape(B, Hq, N, d) if B == 1 else perm

    def gather(self, group=None, async_op: bool = False):
        """In-place all-gather of every rank's chunk (NCCL on GPUs, gloo in the CPU tests)."""
        return dist.all_gather_into_tensor(self.store.view(-1), self.local.reshape(-1), group=group,
                                           async_op=async_op)


def mirror_addresses(buffer_ptrs, rank: int, chunk_offset_bytes: int) -> list[int]:
    """Addresses of this rank's head chunk inside every PEER's full-layer buffer (rank order, self
    excluded): buffer_ptrs[p] is peer p's symmetric buffer as mapped into this device's address space;
    the chunk sits at the same byte offset in every rank's buffer (rank-major storage)."""
    return [int(b) + int(chunk_offset_bytes) for p, b in enumerate(buffer_ptrs) if p != rank]


class PeerHeadOutput:
    """Fused O exchange for KV-head sharding (§8 f2 / §8(e)): the rank-major full-layer O of
    HeadShardedOutput, allocated in symmetric memory (torch.distributed._symmetric_memory maps every
    rank's buffer into every peer's address space over NVLink).  The prefill writes its head chunk into
    its own buffer and, through bfla_sparse_prefill_mirrored, into the same chunk of every peer's
    buffer from the attention epilogue — the exchange rides along tile by tile instead of running as an
    all-gather after the kernel.  finish() is the device-side cross-rank barrier (signal pads) after
    which every rank's buffer holds the whole layer.  Raises if symmetric memory is unavailable (the
    caller then falls back to HeadShardedOutput + NCCL)."""

    def __init__(self, B: int, Hq: int, N: int, d: int, world: int, rank: int, device, group=None,
                 multicast: bool = False):
        import torch.distributed._symmetric_memory as symm

        if Hq % world:
            raise ValueError(f"h_q={Hq} is not divisible by world={world}")
        if world - 1 > 7:
            raise ValueError("at most 7 peers (BFLA_MAX_MIRRORS)")
        self.world, self.rank = world, rank
        self.store = symm.empty((world, B, Hq // world, N, d), dtype=torch.bfloat16, device=device)
        grp = group if group is not None else dist.group.WORLD
        self.hdl = symm.rendezvous(self.store, grp.group_name)
        self.local = self.store[rank]
        base = int(self.hdl.buffer_ptrs[rank])
        off = self.local.data_ptr() - base  # this rank's chunk inside any rank's buffer
        if off < 0:
            raise RuntimeError("symmetric buffer does not start at the tensor")
        self.mirrors = mirror_addresses(self.hdl.buffer_ptrs, rank, off)
        # NVLS (multicast=True): one multimem.st per 16 bytes through the buffer's multicast address
        # reaches every rank's buffer (the switch replicates it) instead of one P2P store per peer
        self.multicast_o = 0
        if multicast:
            mc = int(getattr(self.hdl, "multicast_ptr", 0) or 0)
            if not mc:
                raise RuntimeError("no NVLS multicast address for this symmetric buffer")
            self.multicast_o = mc + off
            self.mirrors = []
        perm = self.store.permute(1, 0, 2, 3, 4)
        self.full = perm.reshape(B, Hq, N, d) if B == 1 else perm

    def finish(self):
        """Every rank's mirrored stores are visible in every buffer once all ranks pass this barrier."""
        self.hdl.barrier(channel=0)


def split_kv_ranges(tkv: int, parts: int) -> list[tuple[int, int]]:
    """Split-KV (§8 f2): `parts` contiguous, equal-width KV-tile ranges [a, b) covering [0, tkv) for
    bfla_sparse_prefill_kvrange; the partials are combined by bfla_merge_partials (LSE merge).  Used
    when one row is too long for one rank (a diffuse head at 32K): its ranges go to different
    GPUs or SMs and only (O_k, LSE_k) travel."""
    edges = [round(k * tkv / parts) for k in range(parts + 1)]
    return [(edges[k], edges[k + 1]) for k in range(parts)]


# ---- §8 f2: split-KV piece planner -------------------------------------------------------------
# A row (r, h, i) of the prefill is ONE work item on ONE SM (its kept tiles run in sequence), so a
# rank's prefill time is about max(its tiles / #SMs, its longest row).  A diffuse head (kappa -> 1)
# has rows of hundreds of kept tiles; at P = 8 one such row outlasts the rank's whole share (DESIGN §8:
# 2.9x of ideal at 32K), and no row partition can fix it.  The planner splits every row longer than
# the per-SM share into KV-tile ranges (bfla_sparse_prefill_kvrange on a row slice), hands the ranges
# of one row to different ranks, balances the remaining rows as contiguous LPT slices around them,
# and the ranges' (O_k, LSE_k) merge with bfla_merge_partials.


def _lpt_rows(counts, nc_tiles: int = 0):
    """Per LPT row rho = (r * h_kv + h) * tq + (tq - 1 - i): kept tiles and causal extent n(i) (tiles)."""
    import numpy as np

    c = np.asarray(counts, dtype=np.int64)
    B, H, tq = c.shape
    kept = c[:, :, ::-1].reshape(-1)  # rho order: descending i inside each (r, h) segment
    i = np.tile(np.arange(tq - 1, -1, -1), B * H)
    a = nc_tiles + 1  # causal tiles of row i: i + a (Eq. 11-13 with N_c a multiple of T)
    return kept, i + a


def plan_pieces(counts, parts: int, row_overhead: int = 3, sms: int = 148, nc_tiles: int = 0,
                max_split: int = 8):
    """Split-KV work plan for `parts` ranks from a host copy of mask.tile_count ([B, h_kv, tq]).

    Returns one list per rank of pieces (rho_begin, rho_end, kv_begin, kv_end, slot): LPT row slice x
    KV-tile range [kv_begin, kv_end) ((0, 0) = the whole row, bfla_sparse_prefill_rows), whose O / LSE
    go to partial buffer `slot` (the merge input; whole rows use slot 0, the k-th range of a split run
    slot k).  Every (row, kept tile) is covered exactly once.  A row is split when its cost (kept tiles
    + row_overhead) exceeds the per-SM share of one rank, ceil(total / parts / sms), together
    with the rest of its head's rows up to the last such row (the longest rows of a head come first in
    rho, so that is one contiguous run per head and one launch per KV range); each run is cut into K <=
    min(parts, max_split) KV ranges of equal estimated work (kept tiles spread uniformly over each row's
    causal extent) and the K pieces go to K different ranks, least loaded first; the other rows are
    then packed as contiguous slices over the ranks in order, minimising the bottleneck (bisection +
    greedy fill around each rank's piece load)."""
    import numpy as np

    kept, ext = _lpt_rows(counts, nc_tiles)
    cost = kept + row_overhead
    nrows = len(cost)
    total = int(cost.sum())
    share = max(row_overhead + 1, -(-total // (parts * sms)))
    heavy = (cost > share) & (kept > 0)
    # one run per (r, h) segment: from the segment's first row (its longest, rho order is descending i)
    # through its last heavy row — each run is ONE launch per KV range, so a rank's pieces never
    # serialise row by row (isolated heavy rows would each cost a launch on a single SM)
    tq = np.asarray(counts).shape[-1]
    for s0 in range(0, nrows, tq):
        hv = np.nonzero(heavy[s0:s0 + tq])[0]
        if len(hv):
            heavy[s0:s0 + hv[-1] + 1] = True
    load = [0.0] * parts
    plan = [[] for _ in range(parts)]
    if not heavy.any():  # nothing to split: the exact bottleneck-optimal row partition
        from . import bfla_balance_rows

        bounds = bfla_balance_rows(np.asarray(counts, dtype=np.int32), parts, row_overhead)
        return [[(bounds[r], bounds[r + 1], 0, 0, 0)] if bounds[r + 1] > bounds[r] else [] for r in range(parts)]
    # heavy runs -> KV-range pieces
    rho = 0
    while rho < nrows:
        if not heavy[rho]:
            rho += 1
            continue
        end = rho
        while end < nrows and heavy[end]:
            end += 1
        # pieces at most half the per-SM share: a piece's longest row is the critical path of its launch
        K = int(min(parts, max_split, -(-2 * int(cost[rho:end].max()) // share)))
        dens = kept[rho:end] / ext[rho:end]  # kept tiles per causal tile of each row
        tkv = int(ext[rho:end].max())
        # work per KV column j: sum over the run's rows that reach j of their density
        col = np.zeros(tkv + 1)
        np.add.at(col, ext[rho:end], -dens)
        col[0] += dens.sum()
        work = np.cumsum(col)[:tkv]
        cum = np.concatenate([[0.0], np.cumsum(work)])
        edges = [0]
        for k in range(1, K):
            e = int(np.searchsorted(cum, cum[-1] * k / K))
            if edges[-1] < e < tkv:
                edges.append(e)
        edges.append(tkv)
        used = set()
        for k in range(len(edges) - 1):
            a_, b_ = edges[k], edges[k + 1]
            pc = float(cum[b_] - cum[a_]) + row_overhead * (end - rho)
            r = min((x for x in range(parts) if x not in used), key=lambda x: load[x])
            used.add(r)
            load[r] += pc
            plan[r].append((rho, end, a_, b_, k))
        rho = end
    # light rows: contiguous slices of the remaining LPT sequence over ranks 0..parts-1
    light = np.nonzero(~heavy)[0]
    lc = cost[light].astype(np.float64)

    pre = np.concatenate([[0.0], np.cumsum(lc)])

    def fill(bound):  # greedy: each rank in order takes the longest prefix that fits its capacity
        cuts, pos = [], 0
        for r in range(parts):
            if r == parts - 1:
                end = len(lc)
            else:
                end = int(np.searchsorted(pre, pre[pos] + bound - load[r] + 1e-9, side="right")) - 1
                end = max(pos, min(end, len(lc)))
            cuts.append((pos, end))
            pos = end
        ok = all(load[r] + pre[b] - pre[a] <= bound + 1e-9 for r, (a, b) in enumerate(cuts))
        return cuts, ok

    lo, hi = max([0.0] + load + ([float(lc.max())] if len(lc) else [])), float(total) + max(load + [0.0])
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if fill(mid)[1]:
            hi = mid
        else:
            lo = mid
    cuts, _ = fill(hi)
    for r, (a, b) in enumerate(cuts):
        if b <= a:
            continue
        seg = light[a:b]
        # contiguous rho runs inside the slice (heavy runs in between were planned above)
        brk = np.nonzero(np.diff(seg) != 1)[0]
        starts = np.concatenate([[0], brk + 1])
        ends = np.concatenate([brk + 1, [len(seg)]])
        for s0, e0 in zip(starts, ends):
            plan[r].append((int(seg[s0]), int(seg[e0 - 1]) + 1, 0, 0, 0))
    return plan


def plan_slots(plan) -> int:
    """Number of partial (O, LSE) buffers a plan writes (1 + the largest KV-range slot)."""
    return 1 + max((p[4] for pl in plan for p in pl), default=0)


def run_plan(problem_for_slot, cfg, mask, pieces, ws=None, stream=None, streams=None) -> None:
    """Enqueue one rank's pieces: whole-row slices through bfla_sparse_prefill_rows, KV-range pieces
    through bfla_sparse_prefill_kvrange; problem_for_slot(k) is the bfla problem whose O / LSE are
    partial buffer k (their LSE must be set: the merge weighs the partials by it).  With `streams`
    (side streams) the pieces are spread over them, forked from and joined back into `stream`, so the
    launches overlap on the GPU (each is one persistent grid; the next fills SMs as the previous drains)
    instead of paying every launch's tail in sequence.  ws is the workspace of a single launch (its item
    counter): concurrent pieces need one workspace each — pass a list."""
    from . import bfla_sparse_prefill_kvrange, bfla_sparse_prefill_rows

    main = torch.cuda.current_stream() if stream is None else stream
    lanes = list(streams) if streams else [main]
    wss = ws if isinstance(ws, (list, tuple)) else [ws] * len(pieces)
    if streams:
        fork = torch.cuda.Event()
        fork.record(main)
        for s_ in lanes:
            s_.wait_event(fork)
    for n, (r0, r1, a, b, slot) in enumerate(pieces):
        st = lanes[n % len(lanes)]
        w = wss[n % len(wss)]
        if a == 0 and b == 0:
            bfla_sparse_prefill_rows(problem_for_slot(slot), cfg, mask, r0, r1, w, st)
        else:
            bfla_sparse_prefill_kvrange(problem_for_slot(slot), cfg, mask, a, b, rows=(r0, r1), ws=w, stream=st)
    if streams:
        for s_ in lanes:
            ev = torch.cuda.Event()
            ev.record(s_)
            main.wait_event(ev)


class PeerFullOutput:
    """Full-layer O in symmetric memory for the cost-balanced mode (§8 f2): every rank's slice writes its
    rows into its own buffer AND, through bfla_sparse_prefill_mirrored, into every peer's buffer at the
    same offsets (P2P TMA stores, or one multimem.st through the NVLS multicast address) — replacing the
    zero-fill + SUM all-reduce.  finish() is the device barrier after which every buffer holds the layer."""

    def __init__(self, shape, world: int, rank: int, device, group=None, multicast: bool = False):
        import torch.distributed._symmetric_memory as symm

        if world - 1 > 7:
            raise ValueError("at most 7 peers (BFLA_MAX_MIRRORS)")
        self.o = symm.empty(tuple(shape), dtype=torch.bfloat16, device=device)
        grp = group if group is not None else dist.group.WORLD
        self.hdl = symm.rendezvous(self.o, grp.group_name)
        off = self.o.data_ptr() - int(self.hdl.buffer_ptrs[rank])
        self.mirrors = mirror_addresses(self.hdl.buffer_ptrs, rank, off)
        self.multicast_o = 0
        if multicast:
            mc = int(getattr(self.hdl, "multicast_ptr", 0) or 0)
            if not mc:
                raise RuntimeError("no NVLS multicast address for this symmetric buffer")
            self.multicast_o = mc + off
            self.mirrors = []

    def finish(self):
        self.hdl.barrier(channel=0)


def request_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Request (batch) slice for request-level sharding: requests are fully independent."""
    per = -(-batch // world)
    return min(batch, rank * per), min(batch, (rank + 1) * per)


# ---- §8 f2: cost-balanced row sharding of the prefill ------------------------------------------
# Head sharding gives every rank h_kv / world heads, but per-head kappa differs (P:443 runs 8 GPUs
# without naming a scheme), so the rank with the densest heads sets the layer time.  Balanced
# sharding keeps Stage 1 + Stage 2 head-sharded (their cost is per head and small), gathers the
# kept-tile lists, and splits the PREFILL by cost: contiguous slices of the LPT row order
# rho = (r * h_kv + h) * Tq + (Tq - 1 - i) whose kept-tile sums are balanced (bfla_balance_rows),
# each run with bfla_sparse_prefill_rows.  The output rows are then assembled across ranks.


def gather_mask_lists(tile_list: torch.Tensor, tile_count: torch.Tensor, batch: int, world: int, group=None):
    """All-gather head-sharded Stage-2 lists into the global layout.

    Local tile_count is [batch, h_kv/world, Tq] and tile_list holds batch * (h_kv/world) * C entries
    (C = causal tiles per (r, h), include/bfla.h); ranks hold consecutive head slices (head_range).
    Returns (tile_list [batch, h_kv * C], tile_count [batch, h_kv, Tq]) — exactly the layout an unsharded
    bfla_expand_rescue writes, because Stage 2 rows are independent and psi takes the global head."""
    out = []
    for t, last in ((tile_list, None), (tile_count, tile_count.shape[-1])):
        t = t.reshape(batch, -1).contiguous()  # per request: [hl * X], head-major
        if dist.get_backend(group) == "nccl":
            buf = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(buf, t, group=group)
        else:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            buf = torch.stack(parts)
        g = buf.permute(1, 0, 2).reshape(batch, -1)  # [B, world * hl * X]: global head order
        out.append(g if last is None else g.reshape(batch, -1, last))
    return out[0], out[1]


def balanced_slice(tile_count_host: torch.Tensor, world: int, rank: int, row_overhead: int = 3) -> tuple[int, int]:
    """This rank's LPT row slice [row_begin, row_end) of a cost-balanced partition (bfla_balance_rows).
    Every rank computes the same bounds from the same gathered counts, so no exchange is needed."""
    from . import bfla_balance_rows

    b = bfla_balance_rows(tile_count_host, world, row_overhead)
    return b[rank], b[rank + 1]


def slice_rows(row_begin: int, row_end: int, h_kv: int, tq: int):
    """(r, h, i) of the LPT rows in a slice, in order (host helper for tests and reports)."""
    out = []
    for rho in range(row_begin, row_end):
        seg, j = divmod(rho, tq)
        out.append((seg // h_kv, seg % h_kv, tq - 1 - j))
    return out


def assemble_rows(o: torch.Tensor, lse: torch.Tensor | None = None, group=None) -> None:
    """Assemble row-sharded outputs in place: every rank zero-filled O (and LSE) before its slice wrote
    its rows, so a SUM all-reduce gives every rank the full output exactly (x + 0 = x).  This is the
    exposed-collective form; the fused form (the epilogue storing O tiles straight into every peer's
    buffer over NVLink multicast) is the f2 follow-up."""
    dist.all_reduce(o, group=group)
    if lse is not None:
        dist.all_reduce(lse, group=group)


class BalancedLayer:
    """One layer of the f2 strong-scaling path on this rank (all buffers on the rank's GPU):

      1. Stage 1 + Stage 2 on the rank's KV-head group (head-sharded views, global psi offset);
      2. all-gather of the kept-tile lists and counts into the full-layer mask layout (NCCL);
      3. cost-balanced LPT row slice from the gathered counts (host, bfla_balance_rows; every rank
         derives the same bounds, so no exchange);
      4. bfla_sparse_prefill_rows over the full layer's Q/K/V for that slice, into a zeroed O;
      5. SUM all-reduce of O (assemble_rows).

    q/k/v are the full layer (head-first, every rank holds them); o is the full-size output."""

    def __init__(self, q, k, v, o, cfg, rank: int, world: int, row_overhead: int = 3, group=None, peer_out=None):
        from . import alloc_mask, alloc_workspace, make_problem

        # peer_out (PeerFullOutput whose .o is `o`): step 4 stores every row into the peers' O as well,
        # step 5 becomes a device barrier — no zero-fill, no all-reduce
        self.peer_out = peer_out

        self.cfg, self.rank, self.world, self.ovh, self.group = cfg, rank, world, row_overhead, group
        self.B, self.Hkv = q.shape[0], k.shape[1]
        # zero-copy strided views of the rank's head group; the shard problem only runs the mask
        # stages, so its O (a view of the full O) is never written through it
        qs, ks, vs, h0 = shard_views(q, k, v, rank, world)
        os_ = shard_views(o, k, v, rank, world)[0]
        self.Ps = make_problem(qs, ks, vs, os_, head_offset=h0)
        self.ms = alloc_mask(self.Ps, cfg)
        self.wss = alloc_workspace(self.Ps, cfg)
        self.o = o
        self.P = make_problem(q, k, v, o)
        self.m = alloc_mask(self.P, cfg)
        self.ws = alloc_workspace(self.P, cfg)
        self.counts_host = torch.empty(self.m.tile_count.shape, dtype=torch.int32).pin_memory()
        self.bounds = None

    def run(self, marks=None, stream=None):
        """One layer; marks (optional) = 4 CUDA events recorded at the stage boundaries
        (start, masks done, lists gathered + sliced, prefill done)."""
        from . import bfla_block_mask, bfla_expand_rescue, bfla_sparse_prefill_mirrored, bfla_sparse_prefill_rows

        st = torch.cuda.current_stream() if stream is None else stream
        rec = (lambda k: marks[k].record(st)) if marks is not None else (lambda k: None)
        # every op of the layer — library calls, collectives, copies, the zero-fill — goes to `st`,
        # so a non-current stream orders them exactly like the current one
        with torch.cuda.stream(st):
            rec(0)
            bfla_block_mask(self.Ps, self.cfg, self.ms, self.wss, st)
            bfla_expand_rescue(self.Ps, self.cfg, self.ms, self.wss, st)
            rec(1)
            tl, tc = gather_mask_lists(self.ms.tile_list, self.ms.tile_count, self.B, self.world, self.group)
            self.m.tile_list[:tl.numel()].copy_(tl.reshape(-1))
            self.m.tile_count.view(tc.shape).copy_(tc)
            self.counts_host.copy_(self.m.tile_count, non_blocking=True)
            st.synchronize()  # the slice bounds are host decisions (a few KB of counts)
            r0, r1 = balanced_slice(self.counts_host.view(self.B, self.Hkv, -1), self.world, self.rank, self.ovh)
            self.bounds = (r0, r1)
            rec(2)
            if self.peer_out is not None:  # fused exchange: the slice's rows land in every rank's O
                if r1 > r0:  # (an empty slice enqueues nothing; rows (0, 0) would mean every row)
                    bfla_sparse_prefill_mirrored(self.P, self.cfg, self.m, self.peer_out.mirrors, rows=(r0, r1),
                                                 ws=self.ws, stream=st, multicast_o=self.peer_out.multicast_o)
                rec(3)
                self.peer_out.finish()
                return
            self.o.zero_()
            bfla_sparse_prefill_rows(self.P, self.cfg, self.m, r0, r1, self.ws, st)
            rec(3)
            assemble_rows(self.o, None, self.group)
