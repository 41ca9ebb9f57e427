"""Summarise an `ncu --set full` report (.ncu-rep) into the per-kernel text kept under profiles/:
time, DRAM bytes, throughput / pipe utilisation, launch shape and the top issue-stall reasons.

usage: python tools/ncu_full_summary.py REPORT.ncu-rep > profiles/rN_ncu_full_TAG.txt"""
import csv
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(out.stdout.splitlines()))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    for r in data:
        print(f"kernel: {r[col['Kernel Name']]}")
        for m in METRICS:
            if m in col and r[col[m]] != "":
                print(f"  {m} = {r[col[m]]} {units[col[m]]}".rstrip())
        stalls = []
        for h, i in col.items():
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len(STALL):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        for v, name in sorted(stalls, reverse=True)[:6]:
            print(f"  stall {name} = {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
