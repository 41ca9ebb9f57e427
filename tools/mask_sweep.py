"""Tab.mask-format sweep: for each BFLA configuration of the
paper's mask table, build the mask on the synthetic Llama-3.1-8B layer (32 Q / 8 KV heads, d = 128,
structured inputs, N = 32K by default) and report tile density (kept / causal, R20), the per-label
split (mass / sink / band / stride / random), the measured mask-build time (Stage 1 + Stage 2,
CUDA events, median) and the sparse prefill time.  The paper's own columns (LongBench on the real
model, A100) are printed beside ours as context only: inputs differ, so densities are not expected to
match.  A keep-ratio sweep (north_star's knob, R9) follows the γ rows.

GPU only:  python tools/mask_sweep.py [--n 32768] [--out profiles/r1_tabmask_sweep.md]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402

# (b, g, gamma, n_local, rho, eta, paper density %, paper mask-build ms) — P:586-600
TAB_MASK = [
    (256, 64, 0.95, 8, 0.0, 0, 8.75, 1.65),
    (256, 64, 0.999, 8, 0.0, 0, 8.85, 1.70),
    (256, 64, 0.95, 8, 0.0, 16, 14.40, 1.78),
    (256, 64, 0.95, 16, 0.0, 16, 16.87, 1.88),
    (256, 64, 0.98, 8, 0.0, 16, 14.62, 1.94),
    (256, 64, 0.99, 8, 0.0, 16, 14.65, 1.76),
    (128, 64, 0.99, 8, 0.1, 16, 20.62, 2.10),
    (256, 64, 0.99, 8, 0.1, 16, 29.57, 2.08),
    (256, 256, 0.99, 8, 0.1, 16, 19.85, 1.72),
    (512, 64, 0.99, 8, 0.1, 16, 28.00, 2.27),
    (512, 128, 0.99, 8, 0.1, 16, 27.32, 2.06),
    (1024, 64, 0.99, 8, 0.1, 16, 43.37, 2.06),
]
LABELS = ["mass", "sink", "band", "stride", "random"]


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def run(prob, cfg, reps):
    o = torch.empty_like(prob.q)
    P = bf.make_problem(prob.q, prob.k, prob.v, o)
    ws = bf.alloc_workspace(P, cfg)
    m = bf.alloc_mask(P, cfg)

    def build():
        bf.bfla_block_mask(P, cfg, m, ws)
        bf.bfla_expand_rescue(P, cfg, m, ws)

    build()
    torch.cuda.synchronize()
    st = m.stats_dict()
    t_mask = timed(build, reps)
    t_attn = timed(lambda: bf.bfla_sparse_prefill(P, cfg, m, ws), reps)
    dens = st["kept_tiles"] / st["causal_tiles"]
    split = [x / st["causal_tiles"] for x in st["label"][1:6]]
    return dens, split, t_mask, t_attn, st["rows_flagged"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/tabmask_sweep.md")
    a = ap.parse_args()
    prob = workloads.structured(303, 1, 32, 8, a.n, a.n, 128, block=256, theta=5e5, device="cuda")
    lines = [f"# Tab.mask sweep — synthetic Llama-3.1-8B layer (32/8 heads, d=128), N={a.n}, structured seed 303, "
             f"B200, T=64, n_sink=1", "",
             "| b | g | γ | n_local | ρ | η | density (ours) | mass / sink / band / stride / random | mask build ms "
             "| sparse prefill ms | flagged rows | paper density (LongBench, A100) | paper build ms (A100) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for b, g, gamma, nl, rho, eta, pd, pms in TAB_MASK:
        cfg = bf.Config(b=b, g=g, T=64, gamma=gamma, n_local=nl, rho=rho, eta=eta)
        try:
            dens, split, tm, ta, fl = run(prob, cfg, a.reps)
            row = (f"| {b} | {g} | {gamma} | {nl} | {rho} | {eta or '—'} | {100 * dens:.2f}% | "
                   + " / ".join(f"{100 * x:.2f}" for x in split) + f" | {tm:.3f} | {ta:.3f} | {fl} | {pd:.2f}% | {pms:.2f} |")
        except Exception as e:  # e.g. G = b/g = 16 not built for FLATTEN
            row = f"| {b} | {g} | {gamma} | {nl} | {rho} | {eta or '—'} | not built: {str(e)[:60]} | | | | | {pd:.2f}% | {pms:.2f} |"
        print(row, flush=True)
        lines.append(row)
    lines += ["", "Keep-ratio selection (R9, north_star knob) at b=256, g=64, n_local=8, η=16, ρ=0:", "",
              "| keep ratio | density | mass / sink / band / stride / random | mask build ms | sparse prefill ms |",
              "|---|---|---|---|---|"]
    for kr in (0.02, 0.05, 0.1, 0.2, 0.4):
        cfg = bf.Config(b=256, g=64, T=64, select=bf.SELECT_RATIO, keep_ratio=kr, n_local=8, eta=16)
        dens, split, tm, ta, _ = run(prob, cfg, a.reps)
        row = (f"| {kr} | {100 * dens:.2f}% | " + " / ".join(f"{100 * x:.2f}" for x in split)
               + f" | {tm:.3f} | {ta:.3f} |")
        print(row, flush=True)
        lines.append(row)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
