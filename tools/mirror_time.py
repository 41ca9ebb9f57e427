"""Cost of the fused O exchange inside the kernel (§8 f2): bfla_sparse_prefill_mirrored with 0, 1, 3
and 7 mirror buffers on ONE GPU (mirrors are local HBM buffers here, so each adds a full O write to HBM;
over NVLink a peer mirror of a head-sharded layer carries 1/P of O).  Prints one JSON line per count.
usage: python tools/mirror_time.py [--workload llama8b-32k] [--reps 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama8b-32k")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
w = WORKLOADS[a.workload]
prob = workloads.structured(303, 1, w["Hq"], w["Hkv"], w["N"], w["N"], w["d"], block=w["b"], theta=w["theta"],
                            device="cuda")
q, k, v = prob.q, prob.k, prob.v
o = torch.empty_like(q)
cfg = bf.Config(b=w["b"], g=w["g"], T=64, gamma=w["gamma"], n_local=w["n_local"], eta=w["eta"], rho=w["rho"])
P = bf.make_problem(q, k, v, o)
ws, m = bf.alloc_workspace(P, cfg), bf.alloc_mask(P, cfg)
bf.bfla_block_mask(P, cfg, m, ws)
bf.bfla_expand_rescue(P, cfg, m, ws)
st = torch.cuda.current_stream()
mirrors_all = [torch.empty_like(q) for _ in range(7)]
for n in (0, 1, 3, 7):
    mir = mirrors_all[:n]
    fn = lambda: bf.bfla_sparse_prefill_mirrored(P, cfg, m, mir, ws=ws)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    ok = all(torch.equal(x, o) for x in mir)
    print(json.dumps({"workload": a.workload, "mirrors": n, "sparse_prefill_ms": ms, "mirrors_equal_local": ok,
                      "extra_o_bytes": n * o.numel() * 2}))
