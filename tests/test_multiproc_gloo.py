"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: KV-head sharding with a global
head_offset reproduces the unsharded mask bit for bit, and the O all-gather assembles head shards in
order.  The per-shard compute here is the oracle (no GPU in this container); the GPU path consumes
exactly the same views, offsets and collective (paper_2605_12193_b200.parallel)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workloads
    from paper_2605_12193_b200 import parallel

    prob = workloads.gaussian(5, 1, 8, 4, 512, 512, 128, sigma=0.8)
    q, k, v, h0 = parallel.shard_views(prob.q, prob.k, prob.v, rank, world)
    f = lambda t: t[0].float().numpy()
    res = oracle.mask_pipeline(f(q), f(k), b=128, g=64, T=64, gamma=0.95, eta=4, rho=0.3, seed=9, head_offset=h0)
    O, _ = oracle.masked_attention(f(q), f(k), f(v), 128 ** -0.5, res["labels"], 64)
    # gather labels and O (as tensors shaped [B=1, heads, ...]) across ranks
    lab = parallel.gather_heads(torch.from_numpy(res["labels"].astype(np.int32))[None], world)
    o_full = parallel.gather_heads(torch.from_numpy(O)[None], world)
    if rank == 0:
        np.save(os.path.join(out_dir, "labels.npy"), lab[0].numpy())
        np.save(os.path.join(out_dir, "o.npy"), o_full[0].numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharding_equals_unsharded(tmp_path, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import workloads

    prob = workloads.gaussian(5, 1, 8, 4, 512, 512, 128, sigma=0.8)
    f = lambda t: t[0].float().numpy()
    full = orc.mask_pipeline(f(prob.q), f(prob.k), b=128, g=64, T=64, gamma=0.95, eta=4, rho=0.3, seed=9)
    O, _ = orc.masked_attention(f(prob.q), f(prob.k), f(prob.v), 128 ** -0.5, full["labels"], 64)
    assert np.array_equal(np.load(tmp_path / "labels.npy"), full["labels"].astype(np.int32))
    assert np.array_equal(np.load(tmp_path / "o.npy"), O)


def test_head_range_and_views():
    from paper_2605_12193_b200 import parallel

    assert [parallel.head_range(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        parallel.head_range(8, 3, 0)
    q = torch.randn(2, 8, 16, 4)
    k = torch.randn(2, 4, 16, 4)
    qs, ks, vs, h0 = parallel.shard_views(q, k, k, 1, 2)
    assert h0 == 2 and qs.shape == (2, 4, 16, 4) and ks.shape == (2, 2, 16, 4)
    assert qs.data_ptr() == q[:, 4].data_ptr()  # zero-copy view
    assert parallel.request_range(5, 2, 1) == (3, 5)


def _worker_balanced(rank, world, port, out_dir):
    """§8 f2 flow on CPU: head-sharded masks -> gathered lists/counts -> cost-balanced row slices ->
    each rank's rows only -> SUM all-reduce.  The per-slice compute is the oracle restricted to the
    slice's rows (the GPU path runs bfla_sparse_prefill_rows on the same slice)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workloads
    from paper_2605_12193_b200 import parallel

    T = 64
    prob = workloads.gaussian(6, 1, 8, 4, 512, 512, 128, sigma=0.8)
    q, k, v, h0 = parallel.shard_views(prob.q, prob.k, prob.v, rank, world)
    f = lambda t: t[0].float().numpy()
    res = oracle.mask_pipeline(f(q), f(k), b=128, g=64, T=T, gamma=0.95, eta=4, rho=0.3, seed=9, head_offset=h0)
    labels = res["labels"]  # [hl, Tq, Tkv]
    hl, tq, tkv = labels.shape
    causal = np.tril(np.ones((tq, tkv), dtype=bool))
    C = int(causal.sum())
    lists = np.full((hl, C), -1, np.int32)
    for h in range(hl):  # compacted rows at the closed-form offsets c_i (include/bfla.h)
        off = 0
        for i in range(tq):
            js = np.nonzero(labels[h, i] > 0)[0]
            lists[h, off:off + len(js)] = js
            off += i + 1
    counts = (labels > 0).sum(-1).astype(np.int32)
    g_list, g_count = parallel.gather_mask_lists(torch.from_numpy(lists).reshape(-1), torch.from_numpy(counts)[None],
                                                 1, world)
    r0, r1 = parallel.balanced_slice(g_count, world, rank)
    # this rank's rows only: the oracle over all heads with the gathered labels, rows outside zeroed
    full_labels = parallel.gather_heads(torch.from_numpy(labels.astype(np.int32))[None], world)[0].numpy()
    O, lse = oracle.masked_attention(f(prob.q), f(prob.k), f(prob.v), 128 ** -0.5, full_labels, T)
    own = np.zeros(O.shape[:2], dtype=bool)
    m = 2  # heads per group (Hq=8, Hkv=4)
    for _, h, i in parallel.slice_rows(r0, r1, 4, tq):
        own[h * m:(h + 1) * m, i * T:(i + 1) * T] = True
    o_t = torch.from_numpy(np.where(own[..., None], O, 0.0))
    l_t = torch.from_numpy(np.where(own, lse, 0.0))
    parallel.assemble_rows(o_t, l_t)
    if rank == 0:
        np.save(os.path.join(out_dir, "list.npy"), g_list[0].numpy().reshape(4, -1))
        np.save(os.path.join(out_dir, "count.npy"), g_count[0].numpy())
        np.save(os.path.join(out_dir, "o.npy"), o_t.numpy())
        np.save(os.path.join(out_dir, "slices.npy"), np.array([r0, r1]))
    dist.barrier()
    dist.destroy_process_group()


def test_balanced_row_sharding_equals_unsharded(tmp_path, orc):
    world = 2
    mp.spawn(_worker_balanced, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import workloads

    prob = workloads.gaussian(6, 1, 8, 4, 512, 512, 128, sigma=0.8)
    f = lambda t: t[0].float().numpy()
    full = orc.mask_pipeline(f(prob.q), f(prob.k), b=128, g=64, T=64, gamma=0.95, eta=4, rho=0.3, seed=9)
    labels = full["labels"]
    counts = (labels > 0).sum(-1)
    assert np.array_equal(np.load(tmp_path / "count.npy"), counts)
    lst = np.load(tmp_path / "list.npy")
    for h in range(labels.shape[0]):
        off = 0
        for i in range(labels.shape[1]):
            assert np.array_equal(lst[h, off:off + counts[h, i]], np.nonzero(labels[h, i] > 0)[0])
            off += i + 1
    O, _ = orc.masked_attention(f(prob.q), f(prob.k), f(prob.v), 128 ** -0.5, labels, 64)
    assert np.array_equal(np.load(tmp_path / "o.npy"), O)
    r0, r1 = np.load(tmp_path / "slices.npy")
    assert r0 == 0 and 0 < r1 < labels.shape[0] * labels.shape[1]


def _worker_gather_b2(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_12193_b200 import parallel

    B, hl, C, Tq = 3, 2, 5, 4
    h = torch.arange(hl) + rank * hl  # global heads of this rank
    lst = (torch.arange(B)[:, None, None] * 1000 + h[None, :, None] * 100 + torch.arange(C)[None, None, :]).int()
    cnt = (torch.arange(B)[:, None, None] * 1000 + h[None, :, None] * 100 + torch.arange(Tq)[None, None, :]).int()
    gl, gc = parallel.gather_mask_lists(lst.reshape(-1), cnt, B, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "gl.npy"), gl.numpy())
        np.save(os.path.join(out_dir, "gc.npy"), gc.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_mask_lists_multi_request(tmp_path):
    """Global layout of the gathered lists with batch > 1: request-major, then global head (the layout
    an unsharded bfla_expand_rescue writes, include/bfla.h)."""
    world = 2
    mp.spawn(_worker_gather_b2, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    B, H, C, Tq = 3, 4, 5, 4
    gl, gc = np.load(tmp_path / "gl.npy"), np.load(tmp_path / "gc.npy")
    want_l = (np.arange(B)[:, None, None] * 1000 + np.arange(H)[None, :, None] * 100 + np.arange(C)).reshape(B, -1)
    want_c = np.arange(B)[:, None, None] * 1000 + np.arange(H)[None, :, None] * 100 + np.arange(Tq)
    assert np.array_equal(gl, want_l) and np.array_equal(gc, want_c)


def _inplace_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workloads
    from paper_2605_12193_b200 import parallel

    prob = workloads.gaussian(6, 1, 8, 4, 384, 384, 128, sigma=0.8)
    q, k, v, h0 = parallel.shard_views(prob.q, prob.k, prob.v, rank, world)
    f = lambda t: t[0].float().numpy()
    res = oracle.mask_pipeline(f(q), f(k), b=128, g=64, T=64, gamma=0.95, eta=4, rho=0.3, seed=9, head_offset=h0)
    O, _ = oracle.masked_attention(f(q), f(k), f(v), 128 ** -0.5, res["labels"], 64)
    out = parallel.HeadShardedOutput(1, 8, 384, 128, world, rank, "cpu", dtype=torch.float64)
    assert out.full.data_ptr() == out.store.data_ptr() and out.full.shape == (1, 8, 384, 128)
    out.local.copy_(torch.from_numpy(O)[None])  # what the prefill kernel writes in place on a GPU
    ptr = out.store.data_ptr()
    out.gather()
    assert out.store.data_ptr() == ptr  # in place: no new buffer
    if rank == 0:
        np.save(os.path.join(out_dir, "o_inplace.npy"), out.full[0].numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharded_output_inplace_gather(tmp_path, orc):
    """The bench's N>1 exchange (parallel.HeadShardedOutput): each rank's head shard is a contiguous
    chunk of the full rank-major O, written in place, and ONE in-place all_gather_into_tensor yields the
    unsharded layer output (world 2, gloo); no staging buffer, no concatenation."""
    world = 2
    mp.spawn(_inplace_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import workloads

    prob = workloads.gaussian(6, 1, 8, 4, 384, 384, 128, sigma=0.8)
    f = lambda t: t[0].float().numpy()
    full = orc.mask_pipeline(f(prob.q), f(prob.k), b=128, g=64, T=64, gamma=0.95, eta=4, rho=0.3, seed=9)
    O, _ = orc.masked_attention(f(prob.q), f(prob.k), f(prob.v), 128 ** -0.5, full["labels"], 64)
    assert np.array_equal(np.load(tmp_path / "o_inplace.npy"), O)


def test_bench_self_launch_command():
    """bench.py --gpus N without torchrun re-launches itself under torch.distributed.run with one rank
    per GPU and a 127.0.0.1 rendezvous (checked on the command it builds, with a stub launcher)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, subprocess; sys.argv=['bench.py','--gpus','4','--steps','2'];"
            "calls=[]; subprocess.call=lambda c: calls.append(c) or 0;"
            "import runpy\ntry:\n runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit as e:\n"
            " assert e.code == 0\nc=calls[0]; print(c)\n"
            "assert c[1:3]==['-m','torch.distributed.run'] and '--nproc-per-node=4' in c and "
            "'--master-addr=127.0.0.1' in c and c[-4:]==['--gpus','4','--steps','2']")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_mirror_addresses_peer_chunks():
    """Fused exchange (parallel.PeerHeadOutput): rank r's head chunk sits at the same byte offset in every
    rank's symmetric buffer; the mirrors are the peers' buffers (self excluded) at that offset, in rank
    order — checked against an explicit rank-major layout."""
    from paper_2605_12193_b200 import parallel

    world, chunk = 4, 3 * 1024
    bases = [0x7f0000000000 + p * (1 << 30) for p in range(world)]  # peer buffers as mapped locally
    for rank in range(world):
        got = parallel.mirror_addresses(bases, rank, rank * chunk)
        assert got == [bases[p] + rank * chunk for p in range(world) if p != rank]
        assert len(got) == world - 1


def test_split_kv_ranges_cover():
    """split_kv_ranges: contiguous, disjoint, covering [0, tkv), widths within one tile of each other."""
    from paper_2605_12193_b200 import parallel

    for tkv, parts in [(512, 3), (64, 8), (7, 4), (2048, 5)]:
        rs = parallel.split_kv_ranges(tkv, parts)
        assert rs[0][0] == 0 and rs[-1][1] == tkv and len(rs) == parts
        assert all(a[1] == b[0] for a, b in zip(rs[:-1], rs[1:]))
        w = [b - a for a, b in rs]
        assert max(w) - min(w) <= 1
