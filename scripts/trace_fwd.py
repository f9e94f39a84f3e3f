"""Read the FM_TRACE clock64 trace of one forward CTA (build: scripts/build_variant.sh trace -DFM_TRACE)."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200", "libflashmask_trace.so")
import numpy as np, torch  # noqa: E402
import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
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
names = ["s0full", "s1full", "p0full", "p1full", "mma_p0", "mma_p1", "mma_s0", "mma_s1", "mma_kf", "s0_xchg",
         "s0_pass1", "prod_K", "s0_pass2", "s0_stw", "prod_V", "mma_vf"]
print("e  " + " ".join(f"{n[:8]:>8s}" for n in names))
for e in range(40):
    print(f"{e:2d} " + " ".join(f"{a[e, s] - t0:8d}" for s in range(len(names))))
print("period", np.median(np.diff(a[5:40, 0])))
