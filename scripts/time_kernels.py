"""Per-kernel timing (CUDA events via the library's timing ABI) for one workload."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = fm.FM_FLAG_DETERMINISTIC if "--det" in sys.argv else 0
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
dev = torch.device("cuda", 0)
tot = {}
F = 0.0
for c in calls:
    x = bench.make_inputs(c, dev)
    ff, fb = bench.effective_flops(c, fm)[:2]
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
    fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], flags=flags)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(True)
    for _ in range(reps):
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
        fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], flags=flags)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    t = fm.flashmask_timing_collect()
    name = c.get("family", "call")
    print(f"{name:24s} fwd {t['fwd'][0]/reps:8.3f} ms ({ff*reps/t['fwd'][0]/1e9:7.1f} TF/s)  "
          f"bwd {t['bwd'][0]/reps:8.3f} ms ({fb*reps/t['bwd'][0]/1e9:7.1f} TF/s)  dq {t['dq'][0]/reps:7.3f} ms  rho {[round(r,3) for r in bench.effective_flops(c, fm)[2]][:4]}",
          flush=True)
