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
