"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of the
path — tensor-core Stage 1 with forced recompute (TMA-staged units), canonical SIMT Stage 1, MEAN,
keep-ratio, per-query-head masks, paged K/V, Stage 2, both attention kernels (d = 128 / 256), dense,
and the row-sliced prefill over a balanced partition (§8 f2).
Run on a GPU box:  compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402

SLACK = 50.0  # bfla_config.certify_slack: widen tau so rows are flagged and the recompute kernels run


def run(prob, cfg, paged=0, slices=0, mirrors=0, seqlens=None, stage1_only=False):
    q, k, v = prob.q.cuda(), prob.k.cuda(), prob.v.cuda()
    o = torch.zeros_like(q)
    lse = torch.zeros(q.shape[:3], dtype=torch.float32, device="cuda")
    if paged:
        kc, vc, pt = workloads.paged(k, v, paged, seed=3, extra_pages=3)
        P = bf.make_problem(q, kc, vc, o, lse, page_table=pt, n_kv=k.shape[2])
    else:
        P = bf.make_problem(q, k, v, o, lse, seqlens=seqlens)
    if cfg is None:
        bf.bfla_prefill(P, None, None, None)
    else:
        ws = bf.alloc_workspace(P, cfg)
        m = bf.alloc_mask(P, cfg, labels=True)
        bf.bfla_block_mask(P, cfg, m, ws)
        if stage1_only:
            torch.cuda.synchronize()
            return o
        bf.bfla_expand_rescue(P, cfg, m, ws)
        if slices:
            bounds = bf.bfla_balance_rows(m.tile_count.cpu(), slices)
            for a, b in zip(bounds[:-1], bounds[1:]):
                bf.bfla_sparse_prefill_rows(P, cfg, m, a, b, ws)
        elif mirrors:  # fused exchange: every O / LSE row also stored into `mirrors` buffers
            mo = [torch.zeros_like(q) for _ in range(mirrors)]
            ml = [torch.zeros_like(lse) for _ in range(mirrors)]
            bf.bfla_sparse_prefill_mirrored(P, cfg, m, mo, ml, ws=ws)
            torch.cuda.synchronize()
            assert all(torch.equal(x, o) for x in mo) and all(torch.equal(x, lse) for x in ml)
        else:
            bf.bfla_sparse_prefill(P, cfg, m, ws)
    torch.cuda.synchronize()
    return o


def main():
    g1 = workloads.gaussian(5, B=1, Hq=8, Hkv=2, Nq=2048, Nkv=2048, d=128, sigma=0.8)
    cases = [
        ("tc scores + recompute", g1, bf.Config(b=256, g=64, eta=4, rho=0.1, certify_slack=SLACK), 0),
        ("keep-ratio", g1, bf.Config(b=256, g=64, select=bf.SELECT_RATIO, keep_ratio=0.2, certify_slack=SLACK), 0),
        ("per-query-head masks", g1, bf.Config(b=256, g=64, mask_groups=bf.MASK_PER_Q_HEAD), 0),
        ("paged", g1, bf.Config(b=256, g=64), 16),
        ("canonical SIMT, ragged chunk", workloads.gaussian(6, B=1, Hq=4, Hkv=1, Nq=1000, Nkv=1500, d=128, sigma=0.8),
         bf.Config(b=128, g=64), 0),
        ("MEAN", g1, bf.Config(b=128, g=64, pool=bf.POOL_MEAN), 0),
        ("d=256", workloads.gaussian(7, B=1, Hq=4, Hkv=2, Nq=1024, Nkv=1024, d=256, sigma=0.8), bf.Config(b=256, g=64), 0),
        ("dense", g1, None, 0),
    ]
    cases = [c + (0,) for c in cases] + [
        ("row slices (3-way balanced), d=128", g1, bf.Config(b=256, g=64), 0, 3),
        ("row slices (5-way balanced), d=256",
         workloads.gaussian(8, B=2, Hq=4, Hkv=2, Nq=1000, Nkv=1000, d=256, sigma=0.8), bf.Config(b=256, g=64), 0, 5),
    ]
    # round 2: tensor-core Stage 1 on ragged N / varlen (+ partial-group fixup), G = 16, g = 1 (any-G
    # canonical kernel), and the mirrored (fused-exchange) epilogues of both attention kernels
    vq = workloads.gaussian(9, B=3, Hq=4, Hkv=2, Nq=1500, Nkv=2600, d=128, sigma=0.8)
    vl = torch.tensor([[1500, 2600], [700, 700], [1100, 1900]], dtype=torch.int32, device="cuda")
    cases += [
        ("ragged tc + fixup", workloads.gaussian(10, B=1, Hq=8, Hkv=2, Nq=2100, Nkv=2100, d=128, sigma=0.8),
         bf.Config(b=256, g=64, eta=4, certify_slack=SLACK), 0, 0),
        ("G=16 (b=1024)", workloads.gaussian(11, B=1, Hq=4, Hkv=2, Nq=3000, Nkv=3000, d=128, sigma=0.8),
         bf.Config(b=1024, g=64), 0, 0),
        ("g=1 any-G canonical", workloads.gaussian(12, B=1, Hq=2, Hkv=1, Nq=600, Nkv=600, d=128, sigma=0.6),
         bf.Config(b=64, g=1), 0, 0),
    ]
    for name, prob, cfg, paged, slices in cases:
        o = run(prob, cfg, paged, slices)
        print(f"{name}: ok, |O| max {o.float().abs().max().item():.3f}", flush=True)
    for name, prob, cfg, kw in [
        ("varlen tc + fixup", vq, bf.Config(b=256, g=64, certify_slack=SLACK), dict(seqlens=vl)),
        ("mirrored d=128 (TMA epilogue)", g1, bf.Config(b=256, g=64), dict(mirrors=2)),
        ("mirrored d=256 (thread stores)", workloads.gaussian(13, B=1, Hq=4, Hkv=2, Nq=1024, Nkv=1024, d=256,
                                                              sigma=0.8), bf.Config(b=256, g=64), dict(mirrors=2)),
        # round 3: score-kernel clusters (multicast B stages, m = 4 -> CTA pairs; m = 1 -> no cluster),
        # split-K finished in the kernel (small grid) and by the reduce kernel (64 tiles x 5 splits)
        ("s1 cluster + in-kernel split finish", workloads.gaussian(14, B=1, Hq=8, Hkv=2, Nq=4096, Nkv=4096, d=128,
                                                                  sigma=0.8), bf.Config(b=256, g=64), dict(stage1_only=True)),
        ("s1 no cluster (m = 1)", workloads.gaussian(15, B=1, Hq=2, Hkv=2, Nq=4096, Nkv=4096, d=128, sigma=0.8),
         bf.Config(b=256, g=64), dict(stage1_only=True)),
        ("s1 cluster + reduce-kernel split finish", workloads.gaussian(16, B=1, Hq=32, Hkv=8, Nq=16384, Nkv=16384,
                                                                      d=128, sigma=0.8), bf.Config(b=256, g=64),
         dict(stage1_only=True)),
    ]:
        o = run(prob, cfg, **kw)
        print(f"{name}: ok, |O| max {o.float().abs().max().item():.3f}", flush=True)


if __name__ == "__main__":
    main()
