"""Time Stage-1/Stage-2 launches with and without the device statistics block (atomic counters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
prob = workloads.structured(303, 1, 32, 8, n, n, 128, block=256, theta=5e5, device="cuda")
o = torch.empty_like(prob.q)
cfg = bf.Config()
P = bf.make_problem(prob.q, prob.k, prob.v, o)
ws = bf.alloc_workspace(P, cfg)
for stats in (True, False):
    m = bf.alloc_mask(P, cfg, stats=stats)
    for _ in range(3):
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tb, tx = [], []
    for _ in range(20):
        e[0].record()
        bf.bfla_block_mask(P, cfg, m, ws)
        e[1].record()
        bf.bfla_expand_rescue(P, cfg, m, ws)
        e[2].record()
        torch.cuda.synchronize()
        tb.append(e[0].elapsed_time(e[1]))
        tx.append(e[1].elapsed_time(e[2]))
    tb.sort()
    tx.sort()
    print(f"n={n} stats={stats}: block_mask {tb[10]:.4f} ms, expand_rescue {tx[10]:.4f} ms")
