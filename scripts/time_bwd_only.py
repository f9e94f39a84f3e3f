"""Per-kernel timing of the backward alone (forward run once up front) — isolates fwd->bwd interactions."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
dev = torch.device("cuda", 0)
for c in calls[:1]:
    x = bench.make_inputs(c, dev)
    ff, fb, _ = bench.effective_flops(c, fm)[:3]
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
    fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"])
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(True)
    for _ in range(reps):
        fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"])
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    t = fm.flashmask_timing_collect()
    print(f"bwd-only {t['bwd'][0]/reps:8.3f} ms ({fb*reps/t['bwd'][0]/1e9:7.1f} TF/s)", flush=True)
    fm.flashmask_timing_enable(True)
    for _ in range(reps):
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    t = fm.flashmask_timing_collect()
    print(f"fwd-only {t['fwd'][0]/reps:8.3f} ms ({ff*reps/t['fwd'][0]/1e9:7.1f} TF/s)", flush=True)
