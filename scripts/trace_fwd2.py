"""Timeline of one K2b CTA pair's leader (build: scripts/build_variant.sh trace2 -DFM_TRACE -DFM_TRACE_BX=<even x>).
Per visited tile e: MMA issue of S_e / PV_e, the softmax of tile e (warpset e % 2) phases, producer loads."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200",
                                           sys.argv[3] if len(sys.argv) > 3 else "libflashmask_trace2.so")
import numpy as np, torch  # noqa: E402
import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 0
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
c = calls[ci]
x = bench.make_inputs(c, torch.device("cuda", 0))
for _ in range(3):
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"], flags=fm.FM_FLAG_FWD_PAIR)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (80 * 16))()
ev = (ctypes.c_longlong * 16)()
fm._lib.flashmask_debug_trace_fwd2(buf, ev)
a = np.array(buf).reshape(80, 16)
e = np.array(ev)
t0 = e[0]
nE = int(e[9])
print(cfg, c.get("family", ci), "nE", nE)
print("events: start 0, list built", e[1] - t0, " Q arrived (MMA)", e[2] - t0, " epilogue", e[3] - t0,
      " epi end", e[4] - t0, " CTA end", e[5] - t0)
names = ["mS_kf", "mS_iss", "mPV_pf", "mPV_iss", "sm_sfull", "sm_p1", "sm_xchg", "sm_chain", "sm_p2done",
         "G_sfull", "G_done", "prod_K", "prod_V", "G_pvpf", "GP_sfull", "GP_done"]
print("e  " + " ".join(f"{n[:9]:>9s}" for n in names))
for i in range(min(nE, 48)):
    g0 = a[0, 9]
    print(f"{i:2d} " + " ".join(f"{a[i, s] - (g0 if s in (9, 10, 13, 14, 15) else t0) if a[i, s] else -1:9d}" for s in range(len(names))))

for r in (64, 65):
    print("tile", r - 44, "per-warp done (ns rel. leader sfull): leader", [int(a[r, k] - a[r - 44, 9]) for k in range(8)],
          " peer", [int(a[r, 8 + k] - a[r - 44, 9]) for k in range(8)], " leader sees p_full", int(a[r - 44, 13] - a[r - 44, 9]))
