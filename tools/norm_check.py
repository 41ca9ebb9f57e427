"""Debug: the fast Stage-1 certification norms (qn, kn in the workspace) against the exact block-max group
norms, per GQA size m and repeat; prints the worst ratios and where they sit (head, block)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2605_12193_b200 as bf  # noqa: E402
import workloads  # noqa: E402
from gpu_util import run_gpu  # noqa: E402
from test_gpu_parity import _ws_norms  # noqa: E402

for m in (1, 2, 4, 8):
    B, Hkv, N, d, b = 1, 2, 20480, 128, 256
    Hq = m * Hkv
    prob = workloads.gaussian(31 + m, B=B, Hq=Hq, Hkv=Hkv, Nq=N, Nkv=N, d=d, sigma=0.8)
    L = N // b
    qx = prob.q[0].float().reshape(Hq, L, b // 64, 64 * d).norm(dim=-1).amax(-1).double().numpy()
    kx = prob.k[0].float().reshape(Hkv, L, b // 64, 64 * d).norm(dim=-1).amax(-1).double().numpy()
    for rep in range(3):
        fast = run_gpu(prob, bf.Config(b=b, g=64, gamma=0.95, scores=bf.SCORES_AUTO), lse=False)
        qn, kn = _ws_norms(fast["ws"], B, Hq, Hkv, N, N, d, b)
        for nm, got, want in (("q", qn[0], qx), ("k", kn[0], kx)):
            r = got / want
            bad = np.argwhere((r > 1 + 2 ** -9) | (r < 1 - 1e-6))
            print(f"m={m} rep={rep} {nm}: ratio min {r.min():.6f} max {r.max():.6f} bad {len(bad)} "
                  f"at {bad[:8].tolist()} vals {[round(float(r[tuple(x)]), 5) for x in bad[:8]]}", flush=True)
