"""Summarise ncu captures into profiles/ (tracked).

    python tools/summarize_ncu.py report <file.ncu-rep> [label]   -> key metrics (text)
    python tools/summarize_ncu.py launches <launches.csv>          -> per-kernel share of device time
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__warps_active.avg.per_cycle_active",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "sm__cycles_active.avg",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def report(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {label or path}"]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"\n## {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                lines.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
    return "\n".join(lines) + "\n"


def launches(path):
    rows = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    reader = csv.DictReader(io.StringIO(text[start:]))
    per = collections.defaultdict(lambda: [0, 0.0])
    unit = ""
    for r in reader:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        per[name][0] += 1
        per[name][1] += v
    total = sum(v for _, v in per.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache serialised): {path}",
             f"total {total:.1f} {unit} over {sum(c for c, _ in per.values())} launches", "",
             "| kernel | launches | total | share |", "|---|---|---|---|"]
    for name, (c, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {name} | {c} | {v:.1f} {unit} | {100 * v / total:.2f}% |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "report":
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""))
    else:
        print(launches(sys.argv[2]))
