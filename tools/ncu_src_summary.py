"""Summarise an `ncu --page source --csv --print-source sass` export: stall samples per opcode and
the hottest instructions.  python tools/ncu_src_summary.py src.csv [--top N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S] or 0) for r in data)
print("total samples", tot)
agg = {}
for r in data:
    op = r[idx["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    s = int(r[S] or 0)
    a = agg.setdefault(o, [0, {}])
    a[0] += s
    for h in stalls:
        v = int(r[idx[h]] or 0)
        if v:
            a[1][h] = a[1].get(h, 0) + v
for o, (s, d) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    top = sorted(d.items(), key=lambda x: -x[1])[:4]
    print(f"{o:14s} {s:7d} {100*s/tot:5.1f}%  " + "  ".join(f"{k[6:]}={v}" for k, v in top))
if "--top" in sys.argv:
    n = int(sys.argv[sys.argv.index("--top") + 1])
    print("\nhottest instructions (row index in the export)")
    for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][S] or 0))[:n]:
        s = int(r[S] or 0)
        d = sorted(((h, int(r[idx[h]] or 0)) for h in stalls), key=lambda x: -x[1])[:3]
        print(f"{i:6d} {s:6d} {r[idx['Source']].strip()[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in d))
