"""SURVEY f2 / paper App. B: forward-only (inference) FlashMask with grouped-query
attention — 32 query heads, 8 key/value heads, d = 128, B = 1 — at N = 8K / 32K / 128K for the
causal-document and share-question families.  Effective TFLOP/s = 4*d*sum(non-SKIP 128x128
tile areas) per query head / K2 time (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
from workloads import masks as wm  # noqa: E402

H, Hkv, d = 32, 8, 128
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
for N in (8192, 32768, 131072):
    for fam in ("causal_document", "share_question", "causal"):
        rng = np.random.default_rng(N)
        m = wm.sample_family(fam, N, rng, (3, 7))
        sri = torch.from_numpy(wm.stack([m], 1)).to(dev)
        g = torch.Generator(device=dev)
        g.manual_seed(N)
        q = torch.randn(1, N, H, d, generator=g, device=dev).to(torch.bfloat16)
        k = torch.randn(1, N, Hkv, d, generator=g, device=dev).to(torch.bfloat16)
        v = torch.randn(1, N, Hkv, d, generator=g, device=dev).to(torch.bfloat16)
        call = dict(masks=[m], causal=m.causal, B=1, N=N, H=H, d=d, heads=range(H), batch_ids=[0])
        ff, _, rho = bench.effective_flops(call, fm)[:3]
        for _ in range(3):
            fm.flashmask_fwd(q, k, v, sri, m.causal)
        torch.cuda.synchronize()
        fm.flashmask_timing_enable(True)
        for _ in range(reps):
            fm.flashmask_fwd(q, k, v, sri, m.causal)
        torch.cuda.synchronize()
        fm.flashmask_timing_enable(False)
        t = fm.flashmask_timing_collect()
        ms = t["fwd"][0] / reps
        tot = sum(v_[0] for v_ in t.values()) / reps
        print(json.dumps({"N": N, "family": fam, "rho_128": round(rho[0], 4), "H": H, "Hkv": Hkv, "d": d,
                          "fwd_ms": round(ms, 4), "fwd_tflops": round(ff / (ms * 1e-3) / 1e12, 1),
                          "call_ms_incl_k1": round(tot, 4)}), flush=True)
