"""Turn scripts/time_kernels.py output (C5 sweep) into a markdown table: per (N, d, family) the
forward / backward / total effective TFLOP/s (skipped tiles excluded, SURVEY d.1) and % of the
measured sustained bf16 peak (MEASURED_PEAKS.json)."""
import json
import os
import re
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
rx = re.compile(r"^(\S+)\s+fwd\s+([\d.]+) ms \(\s*([\d.]+) TF/s\)\s+bwd\s+([\d.]+) ms \(\s*([\d.]+) TF/s\).*rho \[([^\]]*)\]")
print(f"Peak for %: measured sustained bf16 {peak} TF/s (MEASURED_PEAKS.json).\n")
cfg = None
for line in open(sys.argv[1]):
    if line.startswith("== "):
        cfg = line[3:].strip()
        _, N, d = cfg.split(":")
        print(f"\n### N = {N}, d = {d}\n\n| family | rho_128 | fwd TF/s | bwd TF/s | total TF/s | % peak |\n|---|---|---|---|---|---|")
        continue
    m = rx.match(line)
    if m:
        fam, tf_ms, tf, tb_ms, tb, rho = m.groups()
        tf_ms, tf, tb_ms, tb = map(float, (tf_ms, tf, tb_ms, tb))
        tot = (tf * tf_ms + tb * tb_ms) / (tf_ms + tb_ms)
        r = [float(x) for x in rho.split(",")]
        print(f"| {fam} | {sum(r) / len(r):.3f} | {tf:.0f} | {tb:.0f} | {tot:.0f} | {100 * tot / peak:.1f} |")
