"""Summarise ncu reports / launch lists into profiles/<round>/ (run here, no GPU needed)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors_srcunit_tex_op_red.sum", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:70]
        lines.append(f"### {name}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"- {m}: {r[i]} {u[i]}")
    return "\n".join(lines)


def launches(path):
    txt = "".join(l for l in open(path) if not l.startswith("=="))
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = ["| kernel | launches | mean us | share of GPU time |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(lines)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(report(path) if mode == "report" else launches(path))
