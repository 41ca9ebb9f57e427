"""Timeline of the paired-tile attention kernel (k_attn2) from the instrumented build.

Run on a GPU box:  python tools/attn_trace.py [--dense] [--workload llama8b-32k]
(after `python -m paper_2605_12193_b200.build --trace`).  CTAs 0..3 record clock64 stamps per warp
role; this script prints, per role, the mean spacing between events, i.e. where a step's cycles go:

  MMA warp (role 0): 1 K ready, 2 V ready, 3/19 P_q ready (PV issue), 4/20 S_q issued, 5/21 tail PV
  producers (1, 2): 6 K step issued, 7 V step issued
  softmax q (3 + q): 8 S ready, 9 fast pass done, 10/11 P stored (fast / exact), 12 O ready, 13 epilogue done
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402
from paper_2605_12193_b200 import _lib  # noqa: E402

_lib.use_variant("trace")

CTAS, ROLES, NEV = 4, 6, 8192


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--out", default="gpurun_out/attn_trace.json")
    a = ap.parse_args()
    L = _lib.lib()
    assert _lib.LIB_PATH.endswith("libbfla_trace.so"), _lib.LIB_PATH
    N = a.n
    prob = workloads.structured(303, 1, 32, 8, N, N, 128, block=256, theta=5e5, device="cuda")
    o = torch.empty_like(prob.q)
    cfg = bf.Config(b=256, g=64, T=64, gamma=0.99, n_local=8, eta=16, rho=0.0)
    P = bf.make_problem(prob.q, prob.k, prob.v, o)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg)
    buf = torch.zeros(CTAS * ROLES * NEV, dtype=torch.int64, device="cuda")
    L.bfla_debug_set_trace.argtypes = [ctypes.c_void_p]
    bf.bfla_block_mask(P, cfg, m, ws)
    bf.bfla_expand_rescue(P, cfg, m, ws)
    run = (lambda: bf.bfla_prefill(P, None, None, None)) if a.dense else (lambda: bf.bfla_sparse_prefill(P, cfg, m, ws))
    run()
    torch.cuda.synchronize()
    assert L.bfla_debug_set_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    run()
    torch.cuda.synchronize()
    L.bfla_debug_set_trace(ctypes.c_void_p(0))
    raw = buf.view(CTAS, ROLES, NEV).cpu().numpy().view(np.uint64)
    code = (raw >> np.uint64(56)).astype(np.int64)
    t = (raw & np.uint64(0xFFFFFFFFFFFFFF)).astype(np.int64)
    report = {}
    for cta in range(CTAS):
        t0 = min(t[cta, r, 0] for r in range(ROLES) if raw[cta, r, 0])
        for r in range(ROLES):
            n = int((raw[cta, r] != 0).sum())
            c, tt = code[cta, r, :n], t[cta, r, :n] - t0
            # mean gap from event A to the next event B, for each consecutive (A, B) pair kind
            gaps = {}
            for i in range(n - 1):
                key = f"{c[i]}->{c[i + 1]}"
                gaps.setdefault(key, []).append(int(tt[i + 1] - tt[i]))
            report[f"cta{cta}_role{r}"] = {
                "events": n, "span": int(tt[-1] - tt[0]) if n else 0,
                "gaps": {k: [len(v), float(np.mean(v)), float(np.median(v))] for k, v in sorted(gaps.items())}}
        if cta == 0:
            np.savez("gpurun_out/attn_trace_cta0.npz", code=code[0], t=t[0] - t0)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(report, open(a.out, "w"), indent=1)
    for k, v in report.items():
        if k.startswith("cta0") or k.startswith("cta1"):
            print(k, "events", v["events"], "span", v["span"])
            for g, (cnt, mean, med) in v["gaps"].items():
                if cnt >= 4:
                    print(f"   {g:8s} n={cnt:5d} mean={mean:8.0f} median={med:8.0f}")


if __name__ == "__main__":
    main()
