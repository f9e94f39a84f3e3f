"""E3 (paper §5.3, Fig. 4(a), A.4.1 P:556-565): kernel latency vs block sparsity at N = 32K,
H = 32, d = 128, bf16 — SFT-style packed documents in sparsity buckets of width 0.1 (document
masks below 0.5, causal documents above, plus the full mask at 0), one batch entry per bucket.
Reports fwd / bwd / total ms and effective TFLOP/s per bucket and the linear fit of total time
against (1 - rho) (the paper: latency linear in the fraction of visited tiles)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
from workloads import masks as wm  # noqa: E402

N, H, d = 32768, 32, 128
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
rho_fn = bench.rho_gpu(fm)
rows = []
buckets = [None] + [(k / 10, (k + 1) / 10) for k in range(9)]
for bk in buckets:
    if bk is None:
        m = wm.sample_family("full", N, np.random.default_rng(0))
    else:
        m = bench.sft_mask_in_bucket(N, bk[0], bk[1], 7, rho_fn)
    call = dict(masks=[m], causal=m.causal, B=1, N=N, H=H, d=d, heads=range(H), batch_ids=[0])
    x = bench.make_inputs(call, dev)
    ff, fb, rho = bench.effective_flops(call, fm)[:3]
    for _ in range(2):
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], m.causal)
        fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], m.causal)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(True)
    for _ in range(reps):
        o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], m.causal)
        fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], m.causal)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    t = fm.flashmask_timing_collect()
    tf = t["fwd"][0] / reps
    tb = sum(t[k][0] for k in ("bwd_pre", "bwd", "dq_convert")) / reps
    tk = sum(t[k][0] for k in ("expand", "classify")) / reps
    rows.append(dict(bucket=bk, rho=rho[0], fwd_ms=tf, bwd_ms=tb, k1_ms=tk, total_ms=tf + tb + tk,
                     fwd_tf=ff / (tf * 1e-3) / 1e12, bwd_tf=fb / (tb * 1e-3) / 1e12,
                     total_tf=(ff + fb) / ((tf + tb + tk) * 1e-3) / 1e12))
    print(json.dumps(rows[-1]), flush=True)
x1 = np.array([1 - r["rho"] for r in rows])
y = np.array([r["total_ms"] for r in rows])
A = np.vstack([x1, np.ones_like(x1)]).T
coef, res, _, _ = np.linalg.lstsq(A, y, rcond=None)
pred = A @ coef
r2 = 1 - ((y - pred) ** 2).sum() / ((y - y.mean()) ** 2).sum()
print(json.dumps({"fit": "total_ms = a*(1-rho) + b", "a_ms": coef[0], "b_ms": coef[1], "r2": r2}), flush=True)
