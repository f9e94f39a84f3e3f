"""Developer check: run one case through the CUDA path and print errors vs the oracle.
usage: python scripts/dev_check.py <family> <N> <d> [B] [H] [fwd|bwd]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from gpu_util import build_case, oracle_head, to_cuda  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
from workloads import masks as wm  # noqa: E402

fam, N, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
H = int(sys.argv[5]) if len(sys.argv) > 5 else 1
mode = sys.argv[6] if len(sys.argv) > 6 else "bwd"
rng = np.random.default_rng(N + d)
masks = [wm.sample_family(fam, N, rng, (2, 5)) for _ in range(B)]
sri, t = build_case(masks, H, d)
sri_c, tc = to_cuda(sri, t)
causal = masks[0].causal
o, lse = fm.flashmask_fwd(tc["q"], tc["k"], tc["v"], sri_c, causal, out_dtype=torch.float32)
torch.cuda.synchronize()
print("fwd done", flush=True)
if mode == "bwd":
    dq, dk, dv = fm.flashmask_bwd(tc["q"], tc["k"], tc["v"], o, tc["do"], lse, sri_c, causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    print("bwd done", flush=True)
for b in range(B):
    for h in range(H):
        O, L, g = oracle_head(t, masks, sri.numpy(), b, h, 1, causal, with_grad=(mode == "bwd"))
        res = {"O": (o[b, :, h].cpu().numpy(), O)}
        if mode == "bwd":
            res.update({"dQ": (dq[b, :, h].cpu().numpy(), g[0]), "dK": (dk[b, :, h].cpu().numpy(), g[1]),
                        "dV": (dv[b, :, h].cpu().numpy(), g[2])})
        line = [f"b{b}h{h}"]
        for k, (got, ref) in res.items():
            e = np.abs(got - ref)
            bad = np.argwhere(e > 2e-2)
            line.append(f"{k}: max {e.max():.3e} mean {e.mean():.3e} nbad {len(bad)} first {bad[:3].tolist()}")
        Lg = lse[b, h].cpu().numpy()
        fin = np.isfinite(L)
        line.append(f"lse: inf-match {np.array_equal(np.isneginf(Lg), np.isneginf(L))} "
                    f"max {np.abs(Lg[fin] - L[fin]).max() if fin.any() else 0:.3e}")
        print(" | ".join(line), flush=True)
