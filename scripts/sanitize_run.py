"""Small FlashMask workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 (N=128, d=64, fp32 and bf16 inputs), C2-like shapes scaled down (ragged N, d=64/128, GQA,
deterministic dQ), and a back-to-back chain on one stream sharing one workspace (the
programmatic-dependent-launch ordering)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
from workloads import masks as wm  # noqa: E402
from workloads import tensors as wt  # noqa: E402


def run(m, H, d, dtype=torch.bfloat16, Hkv=None, flags=0, ws=None):
    Hkv = Hkv or H
    if getattr(m, "rowwise", False):
        flags |= fm.FM_FLAG_ROWWISE
    sri = torch.from_numpy(wm.stack([m])).cuda()
    q = wt.make_tensor("q", 1, m.N, H, d, dtype=dtype).cuda()
    do = wt.make_tensor("do", 1, m.N, H, d, dtype=dtype).cuda()
    k = wt.make_tensor("k", 1, m.N, Hkv, d, dtype=dtype).cuda()
    v = wt.make_tensor("v", 1, m.N, Hkv, d, dtype=dtype).cuda()
    o, lse = fm.flashmask_fwd(q, k, v, sri, m.causal, flags=flags, workspace=ws, out_dtype=OUT)
    g = fm.flashmask_bwd(q, k, v, o, do, lse, sri, m.causal, flags=flags, workspace=ws)
    return o, lse, g


which = sys.argv[1] if len(sys.argv) > 1 else "all"
# "f32out": fp32 outputs, written by the kernels' own stores (bf16 O / dK / dV leave through TMA
# bulk tensor stores, which initcheck does not track as initialising global memory)
OUT = torch.float32 if "f32out" in sys.argv else None
rng = np.random.default_rng(0)
cases = [
    ("C1 fp32", lambda: run(wm.causal_document([40, 48, 40]), 1, 64, torch.float32)),
    ("C1 bf16", lambda: run(wm.causal_document([40, 48, 40]), 1, 64)),
    ("causal_doc d128 ragged", lambda: run(wm.sample_family("causal_document", 1000, rng, (2, 5)), 2, 128)),
    ("global_sw d64 ragged", lambda: run(wm.sample_family("global_sliding_window", 700, rng, (2, 5)), 2, 64)),
    ("random_eviction d128 det", lambda: run(wm.sample_family("random_eviction", 513, rng, (2, 5)), 2, 128,
                                             flags=fm.FM_FLAG_DETERMINISTIC)),
    ("gqa share_question d64", lambda: run(wm.sample_family("share_question", 640, rng, (2, 5)), 4, 64, Hkv=2)),
    ("rowwise key_window d128", lambda: run(wm.rw_sample_family("key_window", 700, rng, (2, 5)), 2, 128)),
    ("rowwise causal_document d64 det", lambda: run(wm.rw_sample_family("causal_document", 515, rng, (2, 5)), 2, 64,
                                                    flags=fm.FM_FLAG_DETERMINISTIC)),
    ("pair forward causal_document", lambda: run(wm.sample_family("causal_document", 900, rng, (2, 5)), 2, 128,
                                                 flags=fm.FM_FLAG_FWD_PAIR)),
    # R33 bounded single pass (K1e + single-pass K2a + two-pass fixup launch); qk_sparse has fully
    # masked rows, so its units go through the fixup
    ("bounded causal_document d128", lambda: run(wm.sample_family("causal_document", 1000, rng, (2, 5)), 2, 128,
                                                 flags=fm.FM_FLAG_MAX_BOUND)),
    ("bounded qk_sparse d64 fixup", lambda: run(wm.sample_family("qk_sparse", 640, rng, (2, 5)), 2, 64,
                                                flags=fm.FM_FLAG_MAX_BOUND)),
    # 256 forward / 512 backward CTAs: the LPT order (K1d) is used
    ("lpt causal_document 4K x 16 heads", lambda: run(wm.sample_family("causal_document", 4096, rng, (3, 7)), 16, 128)),
]
for name, f in cases:
    if which in ("all", "cases"):
        f()
        torch.cuda.synchronize()
        print("ok", name, flush=True)
if which in ("all", "chain"):
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    ms = [wm.sample_family(f, 768, rng, (2, 5)) for f in ("causal_document", "sliding_window", "document")]
    for i, m in enumerate(ms + ms):
        run(m, 2, 128, ws=ws, flags=fm.FM_FLAG_MAX_BOUND if i % 2 else 0)
    torch.cuda.synchronize()
    print("ok chain", flush=True)
