"""Copy a scripts/gpu_round.sh result (gpurun_out/) into profiles/<round>/ as committed summaries."""
import json
import os
import re
import shutil
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01"
G = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
for f in ("bench_C3", "bench_C2", "bench_C4", "bench_C3_reference"):
    lines = [l for l in open(f"{G}/{f}.json").read().splitlines() if l.strip().startswith("{")]
    open(f"{R}/{f}.json", "w").write(lines[-1] + "\n")
shutil.copy(f"{G}/launches.csv", f"{R}/launches_C3.csv")
hdr = ("Launch list of `python bench.py --steps 2 --warmup 1 --no-e2e --cpu-budget 0.5` under\n"
       "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches:\n"
       "compare SHARES with bench.py's live CUDA-event split, not absolute times).  Raw: launches_C3.csv.\n\n")
run = lambda *a: subprocess.run(["python", "scripts/ncu_summary.py", *a], capture_output=True, text=True).stdout
open(f"{R}/launch_list_C3.md", "w").write(hdr + run("launches", f"{G}/launches.csv"))
for name, rep, note in [
        ("ncu_bwd_summary.md", "prof_bwd", "K4 backward, C3 call (4 x 32 heads, N=32768, d=128), one launch, `ncu --set full --clock-control none`"),
        ("ncu_fwd_summary.md", "prof_fwd", "K2 forward, C3 call, one launch, `ncu --set full --clock-control none`"),
        ("ncu_bwd64_summary.md", "prof_bwd64", "K4 backward at d=64 (C5 N=32768: B=4, H=64, full mask), one launch"),
        ("ncu_k1_summary.md", "prof_k1", "K1a expand / K1b classify, C3"),
        ("ncu_k35_summary.md", "prof_k35", "K3 backward preprocess and K5 dQ convert, C3 (HBM-bound: compare dram bytes / duration with MEASURED_PEAKS hbm_gbs)")]:
    open(f"{R}/{name}", "w").write(note + "\n\n" + run("report", f"{G}/{rep}.ncu-rep"))
if os.path.exists(f"{G}/c5_sweep.txt"):
    sweep = subprocess.run(["python", "scripts/sweep_table.py", f"{G}/c5_sweep.txt"], capture_output=True, text=True).stdout
    open(f"{R}/c5_sweep.md", "w").write(
        "C5 kernel sweep (App. A.5.2 shapes: 128K tokens, hidden 4096), `scripts/time_kernels.py C5:<N>:<d> 3`,\n"
        "CUDA events per kernel; fwd = K2, bwd = K4 (K1/K3/K5 excluded here, included in bench.py lines).\n\n" + sweep)


def metric(path, key):
    m = re.search(re.escape(key) + r": ([\d.]+) Gbyte", open(path).read())
    return float(m.group(1)) * 1e9


bw = metric(f"{R}/ncu_bwd_summary.md", "dram__bytes_read.sum") + metric(f"{R}/ncu_bwd_summary.md", "dram__bytes_write.sum")
fw = metric(f"{R}/ncu_fwd_summary.md", "dram__bytes_read.sum") + metric(f"{R}/ncu_fwd_summary.md", "dram__bytes_write.sum")
json.dump({"config": "C3", "source": f"{R}/ncu_bwd_summary.md, {R}/ncu_fwd_summary.md (ncu --set full --clock-control "
           "none, one launch of the C3 call)", "fm_bwd_kernel_bytes_per_launch": int(bw),
           "fm_fwd_kernel_bytes_per_launch": int(fw)}, open("profiles/traffic_C3.json", "w"), indent=1)
print("saved to", R)
