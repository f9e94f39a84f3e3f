import os, sys, importlib.util
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, numpy as np
import bench
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
def load(lib, tag):
    os.environ["FLASHMASK_LIB"] = os.path.join(ROOT, "paper_2410_01359_b200", lib)
    spec = importlib.util.spec_from_file_location(f"fm_{tag}", os.path.join(ROOT, "paper_2410_01359_b200", "flashmask.py"))
    m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); return m
new, old = load("libflashmask.so", "new"), load("libflashmask_head.so", "old")
calls, _, _ = bench.build_workload("C2", 0, 1, bench.rho_oracle)
dev = torch.device("cuda", 0)
for c in calls:
    x = bench.make_inputs(c, dev)
    res = []
    for m in (new, old, new):
        o, lse = m.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out_dtype=torch.float32)
        g = m.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"], out_dtype=torch.float32)
        torch.cuda.synchronize()
        res.append((o, lse) + tuple(g))
    for name, a, b, a2 in zip(["o", "lse", "dq", "dk", "dv"], res[0], res[1], res[2]):
        fin = torch.isfinite(b)
        d = (a[fin] - b[fin]).abs()
        bad = ((a - b).abs() > 1e-2) & fin
        rows = torch.nonzero(bad.reshape(bad.shape[0], bad.shape[1], -1).any(-1))[:, 1].unique() if bad.any() else []
        print(c["family"], name, "max diff new-old %.3e" % d.max().item(), "new-new %.3e" % (a[fin]-a2[fin]).abs().max().item(),
              "bad rows", list(map(int, rows[:20])) if len(rows) else [], "n", len(rows))
