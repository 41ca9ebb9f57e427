"""Same-box A/B timing of the prefill kernels: masks for a BASELINE workload once, then the sparse
prefill (bfla_sparse_prefill) and the dense comparator (bfla_prefill, config NULL) timed with CUDA
events over --reps launches, plus a bitwise digest of O so variants can be checked for identical
results.  usage: python tools/attn_time.py [--variant NAME] [--workload llama8b-32k] [--reps 20]"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="")
ap.add_argument("--workload", default="llama8b-32k")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--dense", type=int, default=1)
ap.add_argument("--save", default="", help="save a sample of O (every 16th query row) to this .pt file")
ap.add_argument("--compare", default="", help="compare the O sample with this .pt file (max / mean abs diff)")
a = ap.parse_args()
bf._lib.use_variant(a.variant)
w = WORKLOADS[a.workload]
prob = workloads.structured(303, 1, w["Hq"], w["Hkv"], w["N"], w["N"], w["d"], block=w["b"], theta=w["theta"],
                            device="cuda")
q, k, v = prob.q, prob.k, prob.v
o = torch.empty_like(q)
cfg = bf.Config(b=w["b"], g=w["g"], T=64, gamma=w["gamma"], n_local=w["n_local"], eta=w["eta"], rho=w["rho"])
if w["paged"]:
    kc, vc, pt = workloads.paged(k, v, w["paged"], seed=404)
    P = bf.make_problem(q, kc, vc, o, page_table=pt, n_kv=w["N"])
else:
    P = bf.make_problem(q, k, v, o)
ws = bf.alloc_workspace(P, cfg)
m = bf.alloc_mask(P, cfg)
bf.bfla_block_mask(P, cfg, m, ws)
bf.bfla_expand_rescue(P, cfg, m, ws)
st = torch.cuda.current_stream()


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


sp = timed(lambda: bf.bfla_sparse_prefill(P, cfg, m, ws), a.reps)
dig = hashlib.sha1(o.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
sample = o[0, :, ::16].float().cpu()
if a.save:
    torch.save(sample, a.save)
cmp = None
if a.compare and os.path.exists(a.compare):
    ref = torch.load(a.compare)
    dd = (sample - ref).abs()
    cmp = dict(max_abs=float(dd.max()), mean_abs=float(dd.mean()))
st_ = m.stats_dict()
kept = st_["kept_tiles"]
fl = 4 * w["d"] * (w["Hq"] // w["Hkv"]) * 64 * 64 * kept
out = dict(variant=a.variant or "product", workload=a.workload, sparse_ms=sp, sparse_tflops=fl / sp / 1e9,
           kappa=kept / st_["causal_tiles"], o_digest=dig, vs_saved=cmp)
if a.dense:
    Pd = bf.make_problem(q, k, v, o) if not w["paged"] else P
    wsd = bf.alloc_workspace(Pd, None)
    dn = timed(lambda: bf.bfla_prefill(Pd, None, None, wsd), max(2, a.reps // 4))
    N = w["N"]
    out.update(dense_ms=dn, dense_tflops=4 * w["d"] * w["Hq"] * N * (N + 1) / 2 / dn / 1e9)
print(json.dumps(out))
