"""A/B of the f3 refinement in the forward: K2 time with and without FM_FLAG_NO_REFINE on the
PARTIAL-heavy families (C5 shapes), CUDA events through the library's timing API."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in sys.argv[1:] or ["C5:32768:128:qk_sparse,random_eviction,causal_document,causal",
                             "C5:8192:128:qk_sparse,random_eviction,causal_document"]:
    calls, _, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
    for c in calls:
        r = bench.Runner(fm, [c], dev)
        x = r.inputs[0]
        res = {}
        for rep in range(3):
            for name, flags in (("refine", 0), ("no_refine", fm.FM_FLAG_NO_REFINE)):
                o, lse = r.outs[0][0], r.outs[0][1]
                for _ in range(2):
                    fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out=o, lse=lse, flags=flags,
                                     workspace=r.ws_f[0])
                torch.cuda.synchronize()
                fm.flashmask_timing_enable(True, kernels=[fm.FM_KERNEL_FWD, fm.FM_KERNEL_REFINE])
                n = 10
                for _ in range(n):
                    fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], out=o, lse=lse, flags=flags,
                                     workspace=r.ws_f[0])
                torch.cuda.synchronize()
                fm.flashmask_timing_enable(False)
                t = fm.flashmask_timing_collect()
                res.setdefault(name, []).append(t["fwd"][0] / n)
                res.setdefault(name + "_k1c_ms", []).append(t["refine"][0] / n)
        fwd_tf = {k: round(r.F_fwd / (min(v) * 1e-3) / 1e12, 1) for k, v in res.items() if not k.endswith("ms")}
        print(json.dumps({"cfg": cfg.split(":")[:3], "mask": c["family"], "fwd_tflops": fwd_tf,
                          "k1c_ms": round(min(res["refine_k1c_ms"]), 4),
                          "fwd_ms": {k: round(min(v), 3) for k, v in res.items() if not k.endswith("ms")}}), flush=True)
        r.free()
        torch.cuda.empty_cache()
