"""Run the C3 (or given) workload fwd+bwd a few times — a short command for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
flags = int(os.environ.get("FM_PROFILE_FLAGS", "0"))  # e.g. 8 = FM_FLAG_FWD_PAIR
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
dev = torch.device("cuda", 0)
for c in calls:
    x = bench.make_inputs(c, dev)
    for _ in range(reps):
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], flags=flags)
        fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], flags=flags)
torch.cuda.synchronize()
print("done")
