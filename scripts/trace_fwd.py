import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200", "libflashmask_trace.so")
import numpy as np, torch
import bench
from paper_2410_01359_b200 import flashmask as fm
calls, conf, _ = bench.build_workload("C3", 0, 1, bench.rho_gpu(fm))
c = calls[0]
x = bench.make_inputs(c, torch.device("cuda", 0))
for _ in range(2):
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (64 * 16))()
fm._lib.flashmask_debug_trace_fwd.argtypes = [ctypes.c_void_p]
fm._lib.flashmask_debug_trace_fwd(buf)
a = np.array(buf).reshape(64, 16)
t0 = a[0, 8]
names = ["sm0_sfull", "sm1_sfull", "sm0_pfull", "sm1_pfull", "mma_p0", "mma_p1", "mma_s0iss", "mma_s1iss", "mma_kfull", "s0_bar", "s0_p1", "s0_p2beg", "s0_p2end", "s0_stw"]
print("e  " + " ".join(f"{n[:8]:>8s}" for n in names))
for e in range(40):
    print(f"{e:2d} " + " ".join(f"{a[e, s] - t0:8d}" for s in range(14)))
print("period", np.median(np.diff(a[5:40, 0])))
