"""Timeline of one forward CTA (build: scripts/build_variant.sh trace -DFM_TRACE -DFM_TRACE_BX=<x>).
Prints the prologue / Q arrival / per-tile events / epilogue in clocks relative to CTA start."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
os.environ["FLASHMASK_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2410_01359_b200",
                                           sys.argv[3] if len(sys.argv) > 3 else "libflashmask_trace.so")
import numpy as np, torch  # noqa: E402
import bench  # noqa: E402
from paper_2410_01359_b200 import flashmask as fm  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ci = int(sys.argv[2]) if len(sys.argv) > 2 else 0
calls, conf, _ = bench.build_workload(cfg, 0, 1, bench.rho_gpu(fm))
c = calls[ci]
x = bench.make_inputs(c, torch.device("cuda", 0))
for _ in range(3):
    o, lse = fm.flashmask_fwd(x["q"], x["k"], x["v"], x["sri"], c["causal"])
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (64 * 16))()
fm._lib.flashmask_debug_trace_fwd(buf)
ev = (ctypes.c_longlong * 16)()
fm._lib.flashmask_debug_trace_fwd_ev(ev)
a = np.array(buf).reshape(64, 16)
e = np.array(ev)
t0 = e[0]
nE = int(e[9])
print(cfg, c.get("family", ci), "nE", nE)
print("events: start 0, list built", e[1] - t0, " Q arrived (MMA)", e[2] - t0, " epi q0/q1 start", e[3] - t0, e[4] - t0,
      " epi q0/q1 end", e[5] - t0, e[6] - t0, " CTA end", e[7] - t0)
names = ["s0full", "s1full", "p0full", "p1full", "mma_p0", "mma_p1", "mma_s0", "mma_s1", "mma_kf", "s0_xchg",
         "s0_pass1", "prod_K", "s0_pass2", "s0_stw", "prod_V", "mma_vf"]
print("e  " + " ".join(f"{n[:8]:>8s}" for n in names))
for i in range(min(nE, 40)):
    print(f"{i:2d} " + " ".join(f"{a[i, s] - t0 if a[i, s] else -1:8d}" for s in range(len(names))))

bw = (ctypes.c_longlong * (8 * 32))()
if hasattr(fm._lib, "flashmask_debug_trace_fwd_w") and fm._lib.flashmask_debug_trace_fwd_w(bw) == 0:
    w = np.array(bw).reshape(8, 32)
    print("per-warp P-ready (clk, relative to the earliest warp of the tile), entries 20..27; warp w sits on SMSP w % 4")
    for k in range(8):
        for q in range(2):
            ws = w[k, q * 8:(q + 1) * 8]
            if ws.min() > 0:
                print(f"e={20 + k} tile q{q}: " + " ".join(f"w{q * 8 + i}(s{(q * 8 + i) % 4}):{int(ws[i] - ws.min())}" for i in range(8)))
