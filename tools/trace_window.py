"""Print the merged per-role event timeline of CTA 0 around the k-th item boundary (tools/attn_trace.py output)."""
import sys

import numpy as np

z = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace_cta0.npz")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
code, t = z["code"], z["t"]
ev = sorted((t[r][i], r, code[r][i]) for r in range(code.shape[0]) for i in range(code.shape[1]) if code[r][i])
names = {1: "K rdy", 2: "V rdy", 3: "P0 rdy", 19: "P1 rdy", 4: "S0 iss", 20: "S1 iss", 5: "P0last", 21: "P1last",
         15: "Q rdy", 24: "Q wait", 6: "Kload", 7: "Vload", 14: "q_empty", 22: "Q+pref issued", 23: "Q issued", 8: "S rdy",
         16: "ld done", 17: "half0", 9: "exps", 10: "P st", 11: "P st(x)", 12: "O rdy", 13: "epi done", 25: "epi regs+smem", 26: "epi bar", 27: "store read"}
occ = [e for e in ev if e[1] == 3 and e[2] == 12]
t12 = occ[k][0]
for e in ev:
    if t12 - 6000 <= e[0] <= t12 + 12000:
        print(f"{e[0] - t12:7d}  {'MMA KPROD VPROD SMX0 SMX1 QPROD'.split()[e[1]]:6s} {names.get(e[2], e[2])}")
