import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200", "libflashmask_trace.so")
import numpy as np, torch
import bench
from paper_2410_01359_b200 import flashmask as fm
calls, conf, _ = bench.build_workload("C3", 0, 1, bench.rho_gpu(fm))
c = calls[0]
x = bench.make_inputs(c, torch.device("cuda", 0))
o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
for _ in range(2):
    fm.flashmask_bwd(x["q"], x["k"], x["v"], o, x["do"], lse, x["sri"], c["causal"])
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (64 * 16))()
fm._lib.flashmask_debug_trace(buf)
a = np.array(buf).reshape(64, 16)
t0 = a[0, 4]
names = ["mma_top", "mma_sdpfree", "mma_pfull", "mma_dqempty", "c_sfull", "c_computed", "c_pdsfree", "c_dsempty", "c_pfull", "dq_full", "dq_staged", "mma_sdpiss", "mma_gissued", "mma_qissued", "mma_qfull"]
print("t  " + " ".join(f"{n[:9]:>9s}" for n in names))
for t in range(40):
    print(f"{t:2d} " + " ".join(f"{a[t, s] - t0:9d}" for s in range(15)))
d = np.diff(a[5:40, 4])
print("period c_sfull median", np.median(d))
