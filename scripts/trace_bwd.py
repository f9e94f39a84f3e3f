import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200", "libflashmask_trace.so")
import numpy as np, torch
import bench
from paper_2410_01359_b200 import flashmask as fm
calls, conf, _ = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "C3", 0, 1, bench.rho_gpu(fm))
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
names = ["mma_top", "mma_sdpfree", "mma_pfull", "c_dsstored", "c_sfull", "c_computed", "c_pdsfree", "c_dsempty", "c_pfull", "dq_full", "dq_staged", "mma_sdpiss", "mma_gissued", "mma_qissued", "mma_qfull", "c_stwait"]
print("t  " + " ".join(f"{n[:9]:>9s}" for n in names))
for t in range(40):
    print(f"{t:2d} " + " ".join(f"{a[t, s] - t0:9d}" for s in range(16)))
d = np.diff(a[5:40, 4])
print("period c_sfull median", np.median(d))

buf2 = (ctypes.c_longlong * (64 * 16))()
fm._lib.flashmask_debug_trace2(buf2)
a2 = np.array(buf2).reshape(64, 16)
print("per warp (t = 30..39): s_full pass (rel. warp 0) / s_full -> computed / computed -> p_full arrive")
for t in range(30, 40):
    sf = a2[10 + t - 30, :8]; cp = a2[10 + t - 30, 8:16]; pf = a2[t - 30, :8]
    print(t, " ".join(f"w{w}:{int(sf[w]-sf[0])}/{int(cp[w]-sf[w])}/{int(pf[w]-cp[w])}" for w in range(8)))

print("per warp: computed -> ds_empty ok / ds stored / dq_empty ok / p_full arrive (durations)")
for t in range(30, 40):
    cp = a2[10 + t - 30, 8:16]; de = a2[20 + t - 30, :8]; ds = a2[20 + t - 30, 8:16]; dq = a2[30 + t - 30, :8]; pf = a2[t - 30, :8]
    print(t, " ".join(f"w{w}:{int(de[w]-cp[w])}/{int(ds[w]-de[w])}/{int(dq[w]-ds[w])}/{int(pf[w]-dq[w])}" for w in range(8)))
