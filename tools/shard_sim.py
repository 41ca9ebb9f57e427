"""§8 f2 on one GPU: per-rank prefill time of P-way head sharding vs cost-balanced row sharding.

Each rank of a P-GPU strong-scaling run executes one slice of the prefill on a whole GPU, so a
slice's kernel time on this GPU IS that rank's prefill time (the exchange is not modelled).  For
P in {2, 4, 8} this runs every slice of both partitions through bfla_sparse_prefill_rows (CUDA
events, median of --reps after warm-up) and prints one JSON line per (workload, P): per-slice ms,
max over slices (the layer's prefill time at P GPUs), and max / (unsliced / P)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402
from paper_2605_12193_b200 import parallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama8b-32k", choices=list(bench.WORKLOADS))
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--overhead", type=int, default=3, help="per-row cost in tile units (bfla_balance_rows)")
ap.add_argument("--skew", type=int, default=0,
                help="make the first SKEW KV head groups diffuse (Q scaled by 0.05: near-uniform block softmax, "
                     "kappa -> ~1), the dense-head case of real models")
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
N, Hq, Hkv, d = w["N"], w["Hq"], w["Hkv"], w["d"]
prob = bench.make_inputs(w, 303, "cuda")
q, k, v = prob.q, prob.k, prob.v
if a.skew:
    q[:, :a.skew * (Hq // Hkv)] *= 0.05
o = torch.empty_like(q)
cfg = bf.Config(b=w["b"], g=w["g"], T=64, gamma=w["gamma"], n_local=w["n_local"], eta=w["eta"], rho=w["rho"])
if w["paged"]:
    kc, vc, pt = workloads.paged(k, v, w["paged"], seed=404)
    P = bf.make_problem(q, kc, vc, o, page_table=pt, n_kv=N)
else:
    P = bf.make_problem(q, k, v, o)
ws = bf.alloc_workspace(P, cfg)
m = bf.alloc_mask(P, cfg)
bf.bfla_block_mask(P, cfg, m, ws)
bf.bfla_expand_rescue(P, cfg, m, ws)
torch.cuda.synchronize()
counts = m.tile_count.view(1, Hkv, -1).cpu()
Tq = counts.shape[2]
rows = Hkv * Tq


def time_call(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    ts = []
    for _ in range(a.reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def time_slice(r0, r1):
    return time_call(lambda: bf.bfla_sparse_prefill_rows(P, cfg, m, r0, r1, ws))


full = time_slice(0, rows)
kappa_head = [round(float(counts[0, h].sum()) / (Tq * (Tq + 1) / 2), 4) for h in range(Hkv)]
print(json.dumps({"workload": a.workload, "skew": a.skew, "full_ms": round(full, 4), "kappa_per_head": kappa_head}))
for parts in (2, 4, 8):
    if Hkv % parts:
        continue
    res = {}
    # head sharding: rank p runs the whole path on its KV-head group (contiguous copies, global psi)
    t = []
    for p in range(parts):
        qs, ks, vs, h0 = parallel.shard_views(q, k, v, p, parts)
        qs, ks, vs = qs.contiguous(), ks.contiguous(), vs.contiguous()
        os_ = torch.empty_like(qs)
        if w["paged"]:
            kcs, vcs, pts = workloads.paged(ks, vs, w["paged"], seed=404)
            Ps = bf.make_problem(qs, kcs, vcs, os_, page_table=pts, n_kv=N, head_offset=h0)
        else:
            Ps = bf.make_problem(qs, ks, vs, os_, head_offset=h0)
        wss = bf.alloc_workspace(Ps, cfg)
        ms = bf.alloc_mask(Ps, cfg)
        bf.bfla_block_mask(Ps, cfg, ms, wss)
        bf.bfla_expand_rescue(Ps, cfg, ms, wss)
        t.append(time_call(lambda: bf.bfla_sparse_prefill(Ps, cfg, ms, wss)))
        del qs, ks, vs, os_, Ps, wss, ms
    res["heads"] = {"slice_ms": [round(x, 4) for x in t], "max_ms": round(max(t), 4),
                    "max_over_ideal": round(max(t) / (full / parts), 3)}
    bal_b = bf.bfla_balance_rows(counts, parts, a.overhead)
    t = [time_slice(x, y) for x, y in zip(bal_b[:-1], bal_b[1:])]
    res["balanced"] = {"slice_ms": [round(x, 4) for x in t], "max_ms": round(max(t), 4),
                       "max_over_ideal": round(max(t) / (full / parts), 3), "bounds": bal_b}
    # split-KV plan (parallel.plan_pieces): a rank's pieces run back to back on its GPU; the KV-range
    # partials go to slot buffers (the cross-rank merge of the split rows is not timed: one GPU)
    plan = parallel.plan_pieces(counts.numpy(), parts, a.overhead)
    nslot = parallel.plan_slots(plan)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
    o_s = [torch.empty_like(q) for _ in range(nslot)]
    l_s = [torch.empty_like(lse) for _ in range(nslot)]
    if w["paged"]:
        probs = [bf.make_problem(q, kc, vc, o_s[s], l_s[s], page_table=pt, n_kv=N) for s in range(nslot)]
    else:
        probs = [bf.make_problem(q, k, v, o_s[s], l_s[s]) for s in range(nslot)]
    lanes = [torch.cuda.Stream() for _ in range(max(len(pl) for pl in plan))]
    wsl = [ws] + [bf.alloc_workspace(P, cfg) for _ in range(len(lanes) - 1)]  # one item counter per lane
    t = [time_call(lambda pl=pl: parallel.run_plan(lambda s: probs[s], cfg, m, pl, ws=wsl, streams=lanes))
         for pl in plan]
    res["split_kv"] = {"rank_ms": [round(x, 4) for x in t], "max_ms": round(max(t), 4),
                       "max_over_ideal": round(max(t) / (full / parts), 3), "slots": nslot,
                       "kv_pieces": sum(1 for pl in plan for p in pl if p[3])}
    del o_s, l_s, probs
    print(json.dumps({"workload": a.workload, "skew": a.skew, "P": parts, "ideal_ms": round(full / parts, 4), **res}))
