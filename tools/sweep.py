"""SURVEY §8(d) sweeps on one B200 (synthetic `structured` inputs, CUDA events, whole path timed):

  c2  Llama-3.1-8B layer at 32K: gamma in {0.9, 0.95, 0.99, 0.999} x eta in {off, 16}
  c5  Gemma-like global layer (16 Q / 8 KV heads, d = 256): N in {4K ... 128K} x sparsity knobs —
      eta in {off, 32, 16, 8} (rho 0), rho in {0.1, 0.2} (eta 16), keep_ratio in {0.05, 0.1, 0.2, 0.4}
      (--tile 64 or 128)

For every point: kappa (kept / causal tiles, R20), layer ms = Stage 1 + Stage 2 + sparse prefill
(CUDA-graph replays of the captured layer: median with p10 / p90 of --reps layers; inputs exceed L2
from 32K up), the stage split (eager pass),
the dense causal comparator (same kernel, median of 3) and speedup = dense / layer.  Writes a
markdown table and one JSON line per point.

GPU only:  python tools/sweep.py --set c2|c5 [--reps 10] [--out profiles/r1_sweep_c2.md]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402


def pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p * (len(xs) - 1))))]


def run_point(P, cfg, reps):
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for _ in range(2):
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill(P, cfg, m, ws)
    torch.cuda.synchronize()
    tot, s1, s2, at = [], [], [], []
    for _ in range(reps):
        ev[0].record()
        bf.bfla_block_mask(P, cfg, m, ws)
        ev[1].record()
        bf.bfla_expand_rescue(P, cfg, m, ws)
        ev[2].record()
        bf.bfla_sparse_prefill(P, cfg, m, ws)
        ev[3].record()
        torch.cuda.synchronize()
        s1.append(ev[0].elapsed_time(ev[1]))
        s2.append(ev[1].elapsed_time(ev[2]))
        at.append(ev[2].elapsed_time(ev[3]))
        tot.append(ev[0].elapsed_time(ev[3]))
    st = m.stats_dict()
    kappa = st["kept_tiles"] / max(1, st["causal_tiles"])
    # layer time from CUDA-graph replays of the captured layer (no host launch gaps: they dominate
    # below ~8K); the stage split above is from the eager pass
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)
        bf.bfla_sparse_prefill(P, cfg, m, ws)
    graph.replay()
    torch.cuda.synchronize()
    tot = []
    for _ in range(reps):
        ev[0].record()
        graph.replay()
        ev[1].record()
        torch.cuda.synchronize()
        tot.append(ev[0].elapsed_time(ev[1]))
    del graph
    return dict(kappa=kappa, ms=statistics.median(tot), p10=pct(tot, 0.1), p90=pct(tot, 0.9),
                stage1_ms=statistics.median(s1), stage2_ms=statistics.median(s2), prefill_ms=statistics.median(at),
                rows_flagged=st["rows_flagged"])


def dense_ms(P, reps=3):
    wsd = bf.alloc_workspace(P, None)
    bf.bfla_prefill(P, None, None, wsd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        bf.bfla_prefill(P, None, None, wsd)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def layer(Hq, Hkv, d, N, theta, seed):
    prob = workloads.structured(seed, 1, Hq, Hkv, N, N, d, block=256, theta=theta, device="cuda")
    o = torch.empty_like(prob.q)
    return prob, bf.make_problem(prob.q, prob.k, prob.v, o), o


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", choices=["c2", "c5"], required=True)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-n", type=int, default=131072)
    ap.add_argument("--tile", type=int, default=64, choices=[64, 128], help="mask tile T")
    a = ap.parse_args()
    rows = []
    if a.set == "c2":
        prob, P, o = layer(32, 8, 128, 32768, 5e5, 202)
        dm = dense_ms(P)
        for eta in (0, 16):
            for gamma in (0.9, 0.95, 0.99, 0.999):
                cfg = bf.Config(b=256, g=64, T=a.tile, gamma=gamma, n_local=8, eta=eta, rho=0.0)
                r = run_point(P, cfg, a.reps)
                r.update(set="c2", N=32768, knob=f"gamma={gamma} eta={eta or 'off'}", dense_ms=dm,
                         speedup=dm / r["ms"])
                rows.append(r)
                print(json.dumps(r), flush=True)
    else:
        for N in (4096, 8192, 16384, 32768, 65536, 131072):
            if N > a.max_n:
                continue
            prob, P, o = layer(16, 8, 256, N, 1e6, 505)
            dm = dense_ms(P)
            knobs = [(f"eta={e or 'off'}", dict(eta=e, rho=0.0)) for e in (0, 32, 16, 8)]
            knobs += [(f"eta=16 rho={rho}", dict(eta=16, rho=rho)) for rho in (0.1, 0.2)]
            knobs += [(f"keep_ratio={kr}", dict(eta=16, rho=0.0, select=bf.SELECT_RATIO, keep_ratio=kr))
                      for kr in (0.05, 0.1, 0.2, 0.4)]
            for name, kw in knobs:
                cfg = bf.Config(b=256, g=64, T=a.tile, gamma=0.99, n_local=8, **kw)
                r = run_point(P, cfg, a.reps)
                r.update(set="c5", N=N, knob=name, dense_ms=dm, speedup=dm / r["ms"])
                rows.append(r)
                print(json.dumps(r), flush=True)
            del prob, P, o
            torch.cuda.empty_cache()
    lines = [f"# §8(d) sweep {a.set}, T = {a.tile} (B200, synthetic structured inputs; median of {a.reps} layers, "
             "p10/p90)", "",
             "| N | knob | κ | layer ms (p10–p90) | Stage 1 | Stage 2 | prefill | dense ms | speedup | rows flagged |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['N']} | {r['knob']} | {r['kappa']:.4f} | {r['ms']:.3f} ({r['p10']:.3f}–{r['p90']:.3f}) | "
                     f"{r['stage1_ms']:.3f} | {r['stage2_ms']:.3f} | {r['prefill_ms']:.3f} | {r['dense_ms']:.3f} | "
                     f"{r['speedup']:.2f}× | {r['rows_flagged']} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
