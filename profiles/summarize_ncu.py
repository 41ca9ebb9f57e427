#!/usr/bin/env python
"""Summarise ncu reports / launch lists into the small text files committed under profiles/.

  python profiles/summarize_ncu.py rep  <file.ncu-rep>  [out.txt]   # --set full capture -> key metrics
  python profiles/summarize_ncu.py list <launches.csv>  [out.txt]   # gpu__time_duration launch list -> shares
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled",
]


def rep(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:160]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k} = {d[k]} {u.get(k, '')}".rstrip())
        # stall reasons (top 6)
        st = [(h, d[h]) for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        try:
            st = sorted(((float(v.replace(",", "")), h) for h, v in st if v not in ("", "n/a")), reverse=True)[:6]
            for v, h in st:
                out.append(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} = {v:.3f}")
        except ValueError:
            pass
    return "\n".join(out)


def launch_list(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        val = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            val *= 1e3
        elif r["Metric Unit"] == "ms":
            val *= 1e6
        tot[short] = tot.get(short, 0.0) + val
        cnt[short] += 1
    s = sum(tot.values())
    out = [f"{'kernel':92s} {'launches':>8s} {'total_us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"{k:92s} {cnt[k]:8d} {v / 1e3:10.1f} {v / s:7.1%}")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    text = rep(path) if mode == "rep" else launch_list(path)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(text + "\n")
    print(text)
