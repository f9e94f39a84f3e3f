"""K1 (tile classification) HBM microbenchmark — SURVEY d.4: the mask-vector and classification
traffic measured on its own, with per-head masks large enough for a meaningful GB/s
(Hm = 64 heads x N = 128K x C = 4 int32 = 134 MB of startend_row_indices).

K1a reads startend_row_indices (B*Hm*N*C*4 B) and writes the per-tile extrema (B*Hm*Tc*32 B);
K1b reads the extrema and writes the u8 class map (B*Hm*Tr*Tc B) and counts.  Algorithmic bytes
/ mean CUDA-event time (library timing API, on the launch stream); peak = MEASURED_PEAKS hbm_gbs."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
from workloads import masks as wm  # noqa: E402

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
res = []
for (Hm, N, fam) in ((64, 131072, "global_sliding_window"), (1, 131072, "causal_document"), (32, 32768, "document")):
    rng = np.random.default_rng(Hm + N)
    ms = [wm.sample_family(fam, N, rng, (11, 15)) for _ in range(Hm)]
    C = ms[0].C
    sri = torch.from_numpy(np.stack([m.sri for m in ms])[None]).cuda()  # [1, Hm, N, C], one mask per head
    for _ in range(3):
        fm.flashmask_classify(sri, ms[0].causal)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(True)
    for _ in range(reps):
        fm.flashmask_classify(sri, ms[0].causal)
    torch.cuda.synchronize()
    fm.flashmask_timing_enable(False)
    t = fm.flashmask_timing_collect()
    T = -(-N // 128)
    b_exp = Hm * N * C * 4 + Hm * T * 32
    b_cls = Hm * T * 32 + Hm * T * T + Hm * 24
    ms_e, ms_c = t["expand"][0] / reps, t["classify"][0] / reps
    line = {"mask": fam, "Hm": Hm, "N": N, "C": C,
            "K1a_expand": {"us": round(ms_e * 1e3, 2), "bytes": b_exp, "GB/s": round(b_exp / (ms_e * 1e-3) / 1e9, 1),
                           "frac_of_hbm": round(b_exp / (ms_e * 1e-3) / 1e9 / peak, 3)},
            "K1b_classify": {"us": round(ms_c * 1e3, 2), "bytes": b_cls, "GB/s": round(b_cls / (ms_c * 1e-3) / 1e9, 1),
                             "frac_of_hbm": round(b_cls / (ms_c * 1e-3) / 1e9 / peak, 3)},
            "hbm_peak_gbs": peak}
    print(json.dumps(line), flush=True)
