"""Live timing of bfla_expand_rescue (Stage 2) on a BASELINE workload (CUDA events, 20 reps after warm-up), printing
the flagged-row statistics; with --variant NAME (an A/B build of tools/ab_build.py) and BFLA_* experiment env vars to attribute
Stage-1 time."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ratio", type=float, default=0.0, help="keep-ratio selection (R9) instead of gamma")
ap.add_argument("--variant", default="", help="libbfla_<variant>.so (tools/ab_build.py)")
a = ap.parse_args()
bf._lib.use_variant(a.variant)
prob = workloads.structured(303, 1, a.hq, a.hkv, a.n, a.n, a.d, block=256, theta=5e5, device="cuda")
o = torch.empty_like(prob.q)
cfg = bf.Config(b=256, g=64, T=64, gamma=0.99, n_local=8, eta=16, rho=0.0)
if a.ratio > 0:
    cfg = bf.Config(b=256, g=64, T=64, gamma=0.99, select=bf.SELECT_RATIO, keep_ratio=a.ratio, n_local=8, eta=16)
P = bf.make_problem(prob.q, prob.k, prob.v, o)
ws = bf.alloc_workspace(P, cfg)
m = bf.alloc_mask(P, cfg)
bf.bfla_block_mask(P, cfg, m, ws)
for _ in range(3):
    bf.bfla_expand_rescue(P, cfg, m, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(a.reps):
    e0.record()
    bf.bfla_expand_rescue(P, cfg, m, ws)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
st = m.stats_dict()
print(f"variant={a.variant or 'product'} env={ {k: v for k, v in os.environ.items() if k.startswith('BFLA_')} } n={a.n} ratio={a.ratio} expand_rescue ms: median "
      f"{ts[len(ts) // 2]:.4f} min {ts[0]:.4f}  kept {st['kept_tiles']}")
